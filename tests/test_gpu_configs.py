"""Parity for BASELINE.json's configs AS WRITTEN (VERDICT r1 "What's weak" 1-2).

* C0 end to end through the public ``quantized_linear`` against the oracle's
  ``dequantize(Aq) @ dequantize(Wq).T`` (formats.py:424-442) with the oracle's RTN weight
  (quantizers.py:247-255) -- the full problem fits the CPU oracle.
* ``mrfp4_dequantize`` (the full-size checker of test_gpu_fullsize.py) pinned to the oracle's
  ``dequantize``, so a scale-indexing error shared by the checker and K2 cannot cancel out.
* C2: both Llama-3-70B shapes x both formats at full size, M in {1, 16, 128, 512, 2048, 8192}.
  K2 is checked on a random (row, column) sample against the ORACLE computed from the GPU's
  own operand bytes (independent of ``mrfp4_dequantize``), and K1 against the oracle on every
  row when the oracle finishes in seconds (M <= 128), else on a row sample holding the row
  with the tensor's largest rotated magnitude (so the oracle's NVFP4 s_T is the tensor's).
* C3: Qwen3-32B QKV / O / gate-up / down with weights quantized by the REAL reference
  ``mr_gptq(W, H, nvfp4, transform=hadamard(128))`` (gptq.py:274-300) at the layer's full K
  (tests/golden/make_c3.py); the 128-row slice is tiled to the layer's full N.
"""

import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import rotate_f64

pytestmark = pytest.mark.gpu

SPEC = {"mxfp4": P.FormatSpec.mxfp4(), "nvfp4": P.FormatSpec.nvfp4()}
GSZ = {"mxfp4": 32, "nvfp4": 16}
HERE = os.path.dirname(os.path.abspath(__file__))


def rel_fro(y, ref):
    return float(np.linalg.norm(y - ref) / max(np.linalg.norm(ref), 1e-300))


def unswizzle(sf: torch.Tensor, rows: int, sf_cols: int) -> np.ndarray:
    out = torch.empty((rows, sf_cols), dtype=torch.uint8, device=sf.device)
    _lib.check(_lib.lib().mrfp4_sf_unswizzle(_lib.ptr(sf), _lib.ptr(out), rows, sf_cols, _lib.stream_ptr(torch)))
    return out.cpu().numpy()


def oracle_view(codes: torch.Tensor, sf: torch.Tensor, ts: float, rows_sel, fmt: str, K: int, n_rows: int):
    """OracleQuant of rows ``rows_sel`` of a device operand (codes [n_rows, K/2] + swizzled SF)."""
    G = GSZ[fmt]
    sc = unswizzle(sf, n_rows, K // G)[rows_sel]
    c = codes[torch.as_tensor(rows_sel, device=codes.device)].cpu().numpy()
    ec = O.unpack_nibbles(c, len(rows_sel) * K).reshape(len(rows_sel), K)
    return O.OracleQuant(fmt, len(rows_sel), K, G, None, ec, sc, ts, 0.0, 0.0)


# ----------------------------------------------------------------------------- C0
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_c0_quantized_linear_end_to_end_vs_oracle(out_dtype):
    """configs[0]: 16 tokens x q_proj 4096 -> 4096, NVFP4 + H16, RTN weights, online act quant."""
    M, K, N, k = 16, 4096, 4096, 16
    rng = np.random.default_rng(16)
    X = O.bf16_round(rng.standard_normal((M, K)))
    W = O.bf16_round(rng.standard_normal((N, K)) / np.sqrt(K))
    Aq = O.quantize_rtn(X, "nvfp4", hadamard=k)
    Wq = O.quantize_rtn(W, "nvfp4", hadamard=k)
    ref = O.linear_reference(Aq, Wq)
    tr = P.TransformSpec.hadamard(k)
    # weight from the oracle's container (the reference's RTN bytes) and from GPU RTN: same bytes
    w_ref = P.prepare_weight(P.MfpTensor(SPEC["nvfp4"], N, K, Wq.codes.reshape(-1), Wq.scale_codes.reshape(-1),
                                         Wq.tensor_scale, tr, None))
    w_gpu = P.quantize_weight(torch.from_numpy(W).cuda().bfloat16(), SPEC["nvfp4"], tr)
    assert torch.equal(w_gpu.codes, w_ref.codes) and torch.equal(w_gpu.sf, w_ref.sf)
    assert float(w_gpu.tensor_scale_dev.item()) == Wq.tensor_scale
    x = torch.from_numpy(X).cuda().bfloat16()
    for w in (w_ref, w_gpu):
        y = P.quantized_linear(x, w, out_dtype=out_dtype).float().cpu().numpy()
        if out_dtype == torch.float32:
            assert rel_fro(y, ref) <= 1e-5, rel_fro(y, ref)
        else:
            refb = torch.from_numpy(ref).bfloat16().float().numpy()
            assert (np.abs(y - refb) <= np.abs(refb) * 2.0 ** -7 * 1.01 + 1e-30).mean() >= 0.999
            assert rel_fro(y, ref) <= 3e-3
    g = P.GraphedLinear(w_gpu, M, out_dtype=out_dtype)
    yg = g(x).float().cpu().numpy()
    if out_dtype == torch.float32:
        assert rel_fro(yg, ref) <= 1e-5


# ----------------------------------------------------------------------------- dequantize pin
@pytest.mark.parametrize("fmt", ["mxfp4", "nvfp4"])
@pytest.mark.parametrize("rows,cols", [(1, 64), (130, 256), (257, 1024), (128, 4096)])
def test_device_dequantize_matches_oracle(fmt, rows, cols):
    """mrfp4_dequantize == oracle dequantize (formats.py:424-442): exact for MXFP4 (ts * 2^e is
    exact); NVFP4's fp32 ts * dec * v rounds twice, so within 1 fp32 ulp."""
    rng = np.random.default_rng(rows * 7 + cols)
    G = GSZ[fmt]
    ec = rng.integers(0, 16, (rows, cols), dtype=np.uint8)
    sc = rng.integers(100, 150, (rows, cols // G), dtype=np.uint8) if fmt == "mxfp4" else \
        rng.integers(0, 127, (rows, cols // G), dtype=np.uint8)
    ts = float(np.float32(4 / 3)) if fmt == "mxfp4" else float(np.float32(rng.uniform(1e-3, 1e-2)))
    q = O.OracleQuant(fmt, rows, cols, G, None, ec, sc, ts, 0.0, 0.0)
    w = P.prepare_weight(P.MfpTensor(SPEC[fmt], rows, cols, O.pack_nibbles(ec), sc.reshape(-1), ts, None, None))
    out = torch.empty((rows, cols), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().mrfp4_dequantize(_lib.ptr(w.codes), _lib.ptr(w.sf), _lib.ptr(w.tensor_scale_dev), rows,
                                           cols, w.fmt, _lib.ptr(out), _lib.stream_ptr(torch)))
    got = out.cpu().numpy().astype(np.float64)
    ref = O.dequantize(q)
    if fmt == "mxfp4":
        assert np.array_equal(got, ref.astype(np.float32).astype(np.float64))
    else:
        assert np.all(np.abs(got - ref) <= np.abs(ref) * 2.0 ** -23 + 1e-45)


# ----------------------------------------------------------------------------- C2
C2_SHAPES = {"up": (8192, 28672), "down": (28672, 8192)}
C2_K = {"mxfp4": 32, "nvfp4": 16}


@pytest.fixture(scope="module")
def c2_weights():
    cache = {}

    def get(shape, fmt):
        key = (shape, fmt)
        if key not in cache:
            cache.clear()   # one 70B weight resident at a time
            torch.cuda.empty_cache()
            K, N = C2_SHAPES[shape]
            g = torch.Generator(device="cuda").manual_seed(4321)
            W = (torch.randn((N, K), generator=g, device="cuda") / K ** 0.5).bfloat16()
            cache[key] = (P.quantize_weight(W, SPEC[fmt], P.TransformSpec.hadamard(C2_K[fmt])), W)
        return cache[key]
    return get


@pytest.mark.parametrize("M", [1, 16, 128, 512, 2048, 8192])
@pytest.mark.parametrize("fmt", ["nvfp4", "mxfp4"])
@pytest.mark.parametrize("shape", ["up", "down"])
def test_c2_full_size_vs_oracle_sample(shape, fmt, M, c2_weights):
    K, N = C2_SHAPES[shape]
    k = C2_K[fmt]
    w, W = c2_weights(shape, fmt)
    g = torch.Generator(device="cuda").manual_seed(1234 + M)
    x = torch.randn((M, K), generator=g, device="cuda").bfloat16()
    a = P.quantize_rtn(x, SPEC[fmt], transform=P.TransformSpec.hadamard(k))
    y = torch.empty((M, N), dtype=torch.float32, device="cuda")
    P.gemm(a, w, y)
    yb = P.quantized_linear(x, w)             # the public call, bf16 out
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    rng = np.random.default_rng(M + N)
    # --- K1 vs the oracle
    if M <= 128:
        rows = np.arange(M)
    else:
        rows = rng.choice(M, 24, replace=False)
        if fmt == "nvfp4":
            yr = rotate_f64(x, k)
            rows = np.unique(np.append(rows, int(yr.abs().amax(dim=1).argmax())))
            del yr
    Xs = x[torch.from_numpy(rows).cuda()].float().cpu().numpy().astype(np.float64)
    ora = O.quantize_rtn(Xs, fmt, hadamard=k)
    av = oracle_view(a.codes, a.sf, a.tensor_scale, rows, fmt, K, M)
    # north-star bar: >= 99.99% identical (fp32 FWHT vs the reference's fp64 rotation)
    assert (av.element_codes == ora.element_codes).mean() >= 0.9999
    assert (av.scale_codes == ora.scale_codes).mean() >= 0.9999
    assert a.tensor_scale == pytest.approx(ora.tensor_scale, rel=2 ** -22)
    # --- K2 on a (row, column) sample vs the oracle linear of the GPU's operand bytes
    cols = np.sort(rng.choice(N, 256, replace=False))
    wv = oracle_view(w.codes, w.sf, float(w.tensor_scale_dev.item()), cols, fmt, K, N)
    ref = O.linear_reference(av, wv)
    got = y[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy()
    assert rel_fro(got, ref) <= 1e-5, rel_fro(got, ref)
    gotb = yb[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].float().cpu().numpy()
    refb = torch.from_numpy(ref).bfloat16().float().numpy()
    assert (np.abs(gotb - refb) <= np.abs(refb) * 2.0 ** -7 * 1.01 + 1e-30).mean() >= 0.999
    # --- weight RTN bytes vs the oracle on the sampled rows (NVFP4: the oracle needs the whole
    # weight's s_T, which the row holding the largest rotated magnitude carries)
    wrows = cols
    if fmt == "nvfp4":
        wr = rotate_f64(W, k)
        wrows = np.unique(np.append(cols, int(wr.abs().amax(dim=1).argmax())))
        del wr
    wo = O.quantize_rtn(W[torch.from_numpy(wrows).cuda()].float().cpu().numpy().astype(np.float64), fmt, hadamard=k)
    wv2 = oracle_view(w.codes, w.sf, float(w.tensor_scale_dev.item()), wrows, fmt, K, N)
    assert (wv2.element_codes == wo.element_codes).mean() >= 0.9999
    assert (wv2.scale_codes == wo.scale_codes).mean() >= 0.9999
    assert float(w.tensor_scale_dev.item()) == pytest.approx(wo.tensor_scale, rel=2 ** -22)


# ----------------------------------------------------------------------------- C3
C3_FILE = os.path.join(HERE, "golden", "c3_mrgptq.npz")


@pytest.mark.skipif(not os.path.exists(C3_FILE), reason="tests/golden/c3_mrgptq.npz not generated")
@pytest.mark.parametrize("M", [512, 2048])
@pytest.mark.parametrize("layer", ["qkv", "o", "gateup", "down"])
def test_c3_mrgptq_h128_weights_full_size(layer, M):
    """configs[3] as written: reference MR-GPTQ NVFP4 weights with Hadamard-128, the 128-row slice
    tiled to the layer's full N; activations NVFP4 + H128 online."""
    z = np.load(C3_FILE)
    rows, K, N = (int(v) for v in z[f"{layer}_shape"])
    codes, scales, ts = z[f"{layer}_codes"], z[f"{layer}_scales"], float(z[f"{layer}_ts"])
    tr = P.TransformSpec.hadamard(128)
    reps = N // rows
    mfp = P.MfpTensor(SPEC["nvfp4"], N, K, np.tile(codes, reps), np.tile(scales, reps), ts, tr, None)
    w = P.prepare_weight(mfp)
    slice_q = O.OracleQuant("nvfp4", rows, K, 16, 128, O.unpack_nibbles(codes, rows * K).reshape(rows, K),
                            scales.reshape(rows, K // 16), ts, 0.0, 0.0)
    g = torch.Generator(device="cuda").manual_seed(M + K)
    x = torch.randn((M, K), generator=g, device="cuda").bfloat16()
    a = P.quantize_rtn(x, SPEC["nvfp4"], transform=tr)
    y = torch.empty((M, N), dtype=torch.float32, device="cuda")
    P.gemm(a, w, y)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    rng = np.random.default_rng(M * 3 + K)
    rsel = rng.choice(M, 16, replace=False)
    yr = rotate_f64(x, 128)
    rsel = np.unique(np.append(rsel, int(yr.abs().amax(dim=1).argmax())))
    del yr
    ora = O.quantize_rtn(x[torch.from_numpy(rsel).cuda()].float().cpu().numpy().astype(np.float64), "nvfp4",
                         hadamard=128)
    av = oracle_view(a.codes, a.sf, a.tensor_scale, rsel, "nvfp4", K, M)
    assert (av.element_codes == ora.element_codes).mean() >= 0.9999   # NVFP4+H128: s_T may differ 1 ulp
    assert (av.scale_codes == ora.scale_codes).mean() >= 0.9999
    assert a.tensor_scale == pytest.approx(ora.tensor_scale, rel=2 ** -22)
    ref = O.linear_reference(av, slice_q)                    # every slice row against the oracle
    for rep in rng.choice(reps, 3, replace=False):
        got = y[torch.from_numpy(rsel).cuda()][:, rep * rows:(rep + 1) * rows].cpu().numpy()
        assert rel_fro(got, ref) <= 1e-5, rel_fro(got, ref)
