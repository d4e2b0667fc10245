"""Parity at BASELINE.json's full sizes (configs[1]-[4]), where the CPU oracle cannot run the
whole problem:

* K2: the FP4 GEMM (fp32 output) against an fp32 reference matmul of the DEQUANTIZED operands
  computed on the GPU (``mrfp4_dequantize`` + torch fp32, TF32 off) -- the same quantity as
  ``dequantize(Aq) @ dequantize(Wq).T`` (formats.py:424-442); only the summation order differs
  (bar: 1e-5 relative Frobenius, north star 1e-3).
* K1: a row sample of the full activation against the CPU oracle (quantize_rtn,
  quantizers.py:247-255).  MXFP4 scales are row-local; for NVFP4 the sample includes the row
  holding the tensor's largest rotated magnitude, so the oracle's s_T is the full tensor's.
* Determinism: the same inputs give the same bytes.
"""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import act_quant_into, alloc_result, rotate_f64

pytestmark = pytest.mark.gpu

SPEC = {"mxfp4": P.FormatSpec.mxfp4(), "nvfp4": P.FormatSpec.nvfp4()}
SHAPES = {  # BASELINE.json configs: name -> (M, K, N, fmt, k)
    "c1": (2048, 14336, 4096, "mxfp4", 32),
    "c2-up-nv": (2048, 8192, 28672, "nvfp4", 16),
    "c2-down-mx": (2048, 28672, 8192, "mxfp4", 32),
    "c3-gateup": (2048, 5120, 51200, "nvfp4", 128),
    "c4": (8192, 16384, 53248, "nvfp4", 16),
}


def dequant(codes, sf, ts, rows, cols, fmt):
    out = torch.empty((rows, cols), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().mrfp4_dequantize(_lib.ptr(codes), _lib.ptr(sf), _lib.ptr(ts), rows, cols, fmt,
                                           _lib.ptr(out), _lib.stream_ptr(torch)))
    return out


def operands(name, seed=0):
    M, K, N, fmt, k = SHAPES[name]
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((M, K), generator=g, device="cuda").bfloat16()
    W = (torch.randn((N, K), generator=g, device="cuda") / K ** 0.5).bfloat16()
    w = P.quantize_weight(W, SPEC[fmt], P.TransformSpec.hadamard(k))
    return x, w


@pytest.mark.parametrize("name", list(SHAPES))
def test_gemm_full_size_vs_dequantized_fp32(name):
    M, K, N, fmt, k = SHAPES[name]
    x, w = operands(name)
    a = alloc_result(M, K, w.fmt, k, "cuda")
    act_quant_into(x, w.fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    y = torch.empty((M, N), dtype=torch.float32, device="cuda")
    P.gemm(a, w, y)
    da = dequant(a.codes, a.sf, a.tensor_scale_dev, M, K, w.fmt)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        ref = torch.empty((M, N), dtype=torch.float32, device="cuda")
        for n0 in range(0, N, 8192):   # bound the dequantized-weight temporary
            dw = dequant(w.codes[n0:n0 + 8192], w.sf[(n0 // 128) * 512 * (-(-K // (32 if fmt == 'mxfp4' else 16) // 4)):],
                         w.tensor_scale_dev, min(8192, N - n0), K, w.fmt)
            ref[:, n0:n0 + 8192] = da @ dw.T
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    rel = float((y - ref).norm() / ref.norm())
    assert torch.isfinite(y).all()
    assert rel <= 1e-5, rel
    y2 = torch.empty_like(y)
    P.gemm(a, w, y2)
    assert torch.equal(y, y2)


@pytest.mark.parametrize("name", ["c1", "c2-up-nv", "c2-down-mx", "c3-gateup"])
def test_act_quant_full_size_row_sample_vs_oracle(name):
    M, K, N, fmt, k = SHAPES[name]
    x, _ = operands(name, seed=1)
    r = P.quantize_rtn(x, SPEC[fmt], transform=P.TransformSpec.hadamard(k))
    rows = np.random.default_rng(7).choice(M, 48, replace=False)
    if fmt == "nvfp4":   # include the row holding max |rotated x| so the sample's s_T is the tensor's
        y = rotate_f64(x, k)
        rows = np.unique(np.append(rows, int(y.abs().amax(dim=1).argmax())))
    Xs = x[torch.from_numpy(rows).cuda()].float().cpu().numpy().astype(np.float64)
    ora = O.quantize_rtn(Xs, fmt, hadamard=k)
    codes = r.codes[torch.from_numpy(rows).cuda()].cpu().numpy()
    scales = r.scale_codes().cpu().numpy()[rows]
    ec = O.unpack_nibbles(codes, len(rows) * K).reshape(len(rows), K)
    assert (ec == ora.element_codes).mean() >= 0.9999
    assert (scales == ora.scale_codes).mean() >= 0.9999
    assert r.tensor_scale == pytest.approx(ora.tensor_scale, rel=2 ** -22)
    r2 = P.quantize_rtn(x, SPEC[fmt], transform=P.TransformSpec.hadamard(k))
    assert torch.equal(r.codes, r2.codes) and torch.equal(r.sf, r2.sf)
