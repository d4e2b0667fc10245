"""The one-kernel decode linear (mrfp4_linear_decode: act-quant inside the GEMM CTAs, weight on
the 128-row MMA side; K-split clusters, or persistent CTAs for weights wider than one wave) against the oracle's dequantize(Aq) @ dequantize(Wq).T (formats.py:424-442)
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
                                   (24, 256, 128), (1, 16384, 512), (16, 1024, 16384),
                                   # wider than one wave of clusters: the persistent variant
                                   (4, 2048, 24576), (24, 1024, 20480), (16, 4096, 14336),
                                   # two activation segments per thread (M = 17..32)
                                   (24, 4096, 4096), (32, 4096, 2048), (16, 14336, 512)])
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


@pytest.mark.parametrize("fmt,k", [("nvfp4", 64), ("mxfp4", 128), ("nvfp4", 128), ("mxfp4", 64)])
@pytest.mark.parametrize("M,K,N", [(16, 4096, 4096), (3, 2048, 640), (4, 2048, 24576), (16, 4096, 14336)])
def test_decode_large_hadamard(fmt, k, M, K, N):
    """k = 64 / 128: the cross-segment butterfly stages exchange between lanes (both variants)."""
    rng = np.random.default_rng(M + K + N + k)
    X = O.bf16_round(rng.standard_normal((M, K)))
    W = O.bf16_round(rng.standard_normal((N, K)) / np.sqrt(K))
    w = P.quantize_weight(torch.from_numpy(W).cuda().bfloat16(), SPEC[fmt], P.TransformSpec.hadamard(k))
    x = torch.from_numpy(X).cuda().bfloat16()
    assert decode_eligible(M, w, x.dtype)
    y = P.quantized_linear(x, w, out_dtype=torch.float32).cpu().numpy()
    ref = O.linear_reference(O.quantize_rtn(X, fmt, hadamard=k), O.quantize_rtn(W, fmt, hadamard=k))
    assert rel_fro(y, ref) <= 1e-4, rel_fro(y, ref)
    y2 = two_kernel(x, w, torch.float32).cpu().numpy()
    assert rel_fro(y, y2) <= 1e-6


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
    """Shapes the one-kernel path declines (K slices too long for one wave of clusters and an
    activation too large for the persistent variant; M > 32) still run,
    through K1 + K2, with the same result as the explicit two-kernel call."""
    for M, K, N in ((16, 28672, 1024), (48, 2048, 256)):
        w = P.quantize_weight(torch.randn(N, K, device="cuda").bfloat16() / 64, SPEC["mxfp4"],
                              P.TransformSpec.hadamard(32))
        x = torch.randn(M, K, device="cuda").bfloat16()
        assert not decode_eligible(M, w, x.dtype)
        assert torch.equal(P.quantized_linear(x, w), two_kernel(x, w, torch.bfloat16))


E4M3_VALUES = [0.5, 0.625, 0.75, 1.0, 1.125, 1.5, 1.75, 2.0, 2.5, 3.0, 3.5, 4.0, 6.0, 8.0, 12.0, 16.0]
E4M3_POW2 = [0.5, 1.0, 2.0, 4.0, 8.0, 16.0]
E4M3_MIDS = [0.53125, 0.6875, 1.0625, 1.1875, 1.4375, 1.9375, 2.125, 2.375, 3.25, 3.75, 4.25, 6.5, 7.5, 13.0]
FP4_T = [0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0]


def tie_rows(k, M, K, rng):
    """NVFP4 activations built so that s_T = 1 exactly (one |y| = 2688 = 6 * 448) and every
    16-group's scale ratio amax / 6 is an E4M3 value with elements at T * dec for the E2M1
    rounding thresholds T (element ties), or an E4M3 midpoint (scale ties).  k = 0: directly;
    k = 16: each block holds two nonzeros a, b, whose rotation has |y| in {(a+b)/4, |a-b|/4}."""
    X = np.zeros((M, K))
    for r in range(M):
        for g in range(K // 16):
            tie_scale = (r + g) % 2 == 1
            T = rng.choice(FP4_T)
            if k == 0:
                d = rng.choice(E4M3_MIDS if tie_scale else E4M3_VALUES)
                grp = rng.integers(-5, 6, size=16) * d                     # |.| < 6 d, bf16-exact
                if not tie_scale:
                    idx = rng.choice(16, size=7, replace=False)
                    grp[idx] = np.asarray(FP4_T) * d * rng.choice([-1, 1], size=7)
                grp[rng.integers(16)] = 6 * d * rng.choice([-1, 1])
                X[r, 16 * g:16 * g + 16] = grp
            else:
                if tie_scale:   # a + b = 24 M (amax / 6 = M, a midpoint), a - b small
                    m = rng.choice(E4M3_MIDS)
                    q = 2.0 ** (np.floor(np.log2(m)) - 2) * rng.integers(1, 4)
                    a, b = 12 * m + q, 12 * m - q
                else:           # a + b = 24 d (amax = 6 d), a - b = 4 T d (|y| = T d)
                    d = rng.choice(E4M3_POW2)
                    a, b = (12 + 2 * T) * d, (12 - 2 * T) * d
                p0, p1 = rng.choice(16, size=2, replace=False)
                X[r, 16 * g + p0], X[r, 16 * g + p1] = a * rng.choice([-1, 1]), b * rng.choice([-1, 1])
    X[0, :16] = 0.0
    X[0, 0] = 2688.0 * (4 if k == 16 else 1)                         # max |y| = 2688 -> s_T = 1
    assert np.array_equal(O.bf16_round(X), X)
    return X


@pytest.mark.parametrize("k", [0, 16])
def test_decode_exact_on_ties(k):
    """Exact rounding ties everywhere (tie_rows): the decode kernel's division-free re-decisions
    (fma paths, k in {0, 16}) run on thousands of E2M1 / E4M3 midpoints.  K1's codes equal the
    oracle's bit for bit on this input, and the decode output equals the K1 + K2 path's (a
    single code flip would move it by ~1e-3)."""
    rng = np.random.default_rng(100 + k)
    M, K, N, fmt = 16, 4096, 1024, "nvfp4"
    X = tie_rows(k, M, K, rng)
    Aq = O.quantize_rtn(X, fmt, hadamard=k or None)
    assert Aq.tensor_scale == 1.0
    Y = O.rotate_blockwise(X, k or None)
    amax = np.abs(Y.reshape(M, -1, 16)).max(axis=2)
    assert np.isin(amax / 6, E4M3_MIDS).sum() > 1000                      # scale ties
    u = np.abs(Y.reshape(M, -1, 16)) / O.E4M3_LEVELS[Aq.scale_codes.astype(int)][:, :, None]
    assert np.isin(u, FP4_T).sum() > 1000                                  # element ties
    W = O.bf16_round(rng.standard_normal((N, K)) / np.sqrt(K))
    tr = P.TransformSpec.hadamard(k) if k else None
    w = P.quantize_weight(torch.from_numpy(W).cuda().bfloat16(), SPEC[fmt], tr)
    x = torch.from_numpy(X).cuda().bfloat16()
    assert decode_eligible(M, w, x.dtype)
    a = alloc_result(M, K, w.fmt, w.had_k, x.device)
    act_quant_into(x, w.fmt, w.had_k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    codes = O.unpack_nibbles(a.codes.cpu().numpy(), M * K).reshape(M, K)
    from paper_2509_23202_b200 import _lib
    sf = torch.empty((M, K // 16), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().mrfp4_sf_unswizzle(_lib.ptr(a.sf), _lib.ptr(sf), M, K // 16, _lib.stream_ptr(torch)))
    assert np.array_equal(sf.cpu().numpy(), Aq.scale_codes.reshape(M, K // 16))
    assert np.array_equal(codes, Aq.element_codes.reshape(M, K))
    y = P.quantized_linear(x, w, out_dtype=torch.float32).cpu().numpy()
    y2 = two_kernel(x, w, torch.float32).cpu().numpy()
    assert rel_fro(y, y2) <= 1e-6
