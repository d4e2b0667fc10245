"""The one-kernel decode linear (mrfp4_linear_decode: act-quant inside the GEMM CTAs, weight on
the 128-row MMA side) against the oracle's dequantize(Aq) @ dequantize(Wq).T (formats.py:424-442)
and against the two-kernel path (K1 + K2) it replaces for M <= 32."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2509_23202_b200 as P
from paper_2509_23202_b200.linear import decode_eligible
from paper_2509_23202_b200.quantize import act_quant_into, alloc_result

pytestmark = pytest.mark.gpu

SPEC = {"mxfp4": P.FormatSpec.mxfp4(), "nvfp4": P.FormatSpec.nvfp4()}


def rel_fro(y, ref):
    return float(np.linalg.norm(y - ref) / max(np.linalg.norm(ref), 1e-300))


def two_kernel(x, w, out_dtype):
    M, K = x.shape
    a = alloc_result(M, K, w.fmt, w.had_k, x.device)
    act_quant_into(x, w.fmt, w.had_k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    y = torch.empty((M, w.N), dtype=out_dtype, device=x.device)
    P.gemm(a, w, y)
    return y


@pytest.mark.parametrize("fmt,k", [("nvfp4", 16), ("mxfp4", 32), ("nvfp4", 32), ("mxfp4", 16), ("nvfp4", 0),
                                   ("mxfp4", 0)])
@pytest.mark.parametrize("M,K,N", [(16, 4096, 4096), (1, 4096, 1024), (7, 2048, 384), (32, 4096, 1024),
                                   (24, 256, 128), (1, 16384, 512), (16, 1024, 16384)])
def test_decode_kernel_vs_oracle_and_two_kernel_path(fmt, k, M, K, N):
    rng = np.random.default_rng(M * 7 + K + N + k)
    X = O.bf16_round(rng.standard_normal((M, K)) * np.exp(rng.uniform(-1, 1, size=(M, 1))))
    W = O.bf16_round(rng.standard_normal((N, K)) / np.sqrt(K))
    tr = P.TransformSpec.hadamard(k) if k else None
    w = P.quantize_weight(torch.from_numpy(W).cuda().bfloat16(), SPEC[fmt], tr)
    x = torch.from_numpy(X).cuda().bfloat16()
    assert decode_eligible(M, w, x.dtype)
    y = P.quantized_linear(x, w, out_dtype=torch.float32).cpu().numpy()
    ref = O.linear_reference(O.quantize_rtn(X, fmt, hadamard=k or None), O.quantize_rtn(W, fmt, hadamard=k or None))
    # north-star bar (1e-3); the rare rotation-rounding code flips of K1 (>= 99.99% identical codes)
    # put the fp32 result at <= 1e-4 here, and the fused kernel equals the two-kernel path below
    assert rel_fro(y, ref) <= 1e-4, rel_fro(y, ref)
    y2 = two_kernel(x, w, torch.float32).cpu().numpy()
    assert rel_fro(y, y2) <= 1e-6
    yb = P.quantized_linear(x, w)                                  # bf16 output: the same fp32
    assert torch.equal(yb.cpu(), torch.from_numpy(y).bfloat16())   # accumulators, rounded once (RNE)
    y3 = P.quantized_linear(x, w, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(y, y3)                                   # deterministic split-K order


@pytest.mark.parametrize("fmt,k", [("nvfp4", 16), ("mxfp4", 32)])
def test_graphed_decode_matches_eager(fmt, k):
    rng = np.random.default_rng(5)
    M, K, N = 16, 4096, 4096
    W = O.bf16_round(rng.standard_normal((N, K)) / 64)
    w = P.quantize_weight(torch.from_numpy(W).cuda().bfloat16(), SPEC[fmt], P.TransformSpec.hadamard(k))
    g = P.GraphedLinear(w, M)
    assert g.decode
    for seed in range(3):
        X = torch.from_numpy(O.bf16_round(np.random.default_rng(seed).standard_normal((M, K)))).cuda().bfloat16()
        y = g(X).clone()
        torch.cuda.synchronize()
        assert torch.equal(y, P.quantized_linear(X, w))


def test_decode_nonfinite_raises():
    w = P.quantize_weight(torch.randn(256, 1024, device="cuda").bfloat16() / 32, SPEC["nvfp4"],
                          P.TransformSpec.hadamard(16))
    x = torch.randn(4, 1024, device="cuda").bfloat16()
    x[1, 7] = float("nan")
    with pytest.raises(P.DataError):
        P.quantized_linear(x, w, check=True)


def test_non_decode_shapes_fall_back_to_two_kernels():
    """Shapes the one-kernel path declines (a per-CTA slice over 16K elements, M > 32) still run,
    through K1 + K2, with the same result as the explicit two-kernel call."""
    for M, K, N in ((16, 14336, 512), (48, 2048, 256)):
        w = P.quantize_weight(torch.randn(N, K, device="cuda").bfloat16() / 64, SPEC["mxfp4"],
                              P.TransformSpec.hadamard(32))
        x = torch.randn(M, K, device="cuda").bfloat16()
        assert not decode_eligible(M, w, x.dtype)
        assert torch.equal(P.quantized_linear(x, w), two_kernel(x, w, torch.bfloat16))
