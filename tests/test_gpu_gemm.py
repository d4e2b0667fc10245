"""K2 parity: tcgen05 block-scaled FP4 GEMM vs the oracle's dequantize-matmul.

Oracle: ``dequantize(A) @ dequantize(W).T`` (formats.py:424-442) computed here in
float64 from the same codes/scales.  Tolerance (north star): relative Frobenius
error <= 1e-3; measured in fp32-output mode where only accumulation order differs
(we assert <= 1e-5).  bf16 output is checked against bf16(Y_ref) to within one
bf16 ulp per element (bf16 rounding alone is 1.66e-3 Frobenius).
"""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2509_23202_b200 as P

pytestmark = pytest.mark.gpu

SPEC = {"mxfp4": P.FormatSpec.mxfp4(), "nvfp4": P.FormatSpec.nvfp4()}


def random_container(rng, rows, cols, fmt, ts=None):
    """Random valid codes/scales as an oracle-style quantization (no data needed)."""
    G = 32 if fmt == "mxfp4" else 16
    ec = rng.integers(0, 16, (rows, cols), dtype=np.uint8)
    if fmt == "mxfp4":
        sc = rng.integers(120, 135, (rows, cols // G), dtype=np.uint8)
        ts = float(np.float32(4 / 3)) if ts is None else ts
    else:
        sc = rng.integers(1, 127, (rows, cols // G), dtype=np.uint8)
        ts = float(np.float32(rng.uniform(0.001, 0.01))) if ts is None else ts
    return O.OracleQuant(fmt, rows, cols, G, None, ec, sc, ts, 0.0, 0.0)


def to_mfp(q):
    return P.MfpTensor(SPEC[q.fmt], q.rows, q.cols, O.pack_nibbles(q.element_codes), q.scale_codes.reshape(-1),
                       q.tensor_scale, None, None)


def run_gemm(A, W, out_dtype=torch.float32):
    a = P.prepare_weight(to_mfp(A))       # same device layout for activations
    w = P.prepare_weight(to_mfp(W))
    act = P.GpuQuantResult(a.fmt, a.N, a.K, 0, a.codes, a.sf, a.tensor_scale_dev,
                           torch.zeros(12, dtype=torch.int32, device="cuda"))
    out = torch.empty((A.rows, W.rows), dtype=out_dtype, device="cuda")
    P.gemm(act, w, out)
    torch.cuda.synchronize()
    return out


def ref64(A, W):
    return O.dequantize(A) @ O.dequantize(W).T


def rel_fro(y, ref):
    return float(np.linalg.norm(y - ref) / max(np.linalg.norm(ref), 1e-300))


@pytest.fixture(params=[1, 2], ids=["cta1", "cta2"])
def kernel(request):
    """Force the 1-CTA or the 2-CTA (cta_group::2) GEMM kernel for this test."""
    import ctypes
    from paper_2509_23202_b200 import _lib
    fn = _lib.lib().mrfp4_debug_gemm_kernel
    fn.argtypes = [ctypes.c_int]
    old = fn(request.param)
    yield request.param
    fn(old)


@pytest.mark.parametrize("fmt", ["mxfp4", "nvfp4"])
@pytest.mark.parametrize("M,N,K", [
    (128, 256, 256), (1, 256, 64), (16, 512, 4096), (200, 384, 1024), (300, 264, 192), (512, 1024, 2048),
    (640, 768, 1280)])
def test_gemm_random_codes_fp32(fmt, M, N, K, kernel):
    rng = np.random.default_rng(M * 131 + N * 7 + K)
    A, W = random_container(rng, M, K, fmt), random_container(rng, N, K, fmt)
    y = run_gemm(A, W).cpu().numpy()
    ref = ref64(A, W)
    assert np.isfinite(y).all()
    assert rel_fro(y, ref) <= 1e-5, rel_fro(y, ref)


@pytest.mark.parametrize("fmt", ["mxfp4", "nvfp4"])
@pytest.mark.parametrize("M,N,K,dtype", [
    (16, 4096, 4096, torch.float32), (16, 4096, 4096, torch.bfloat16), (1, 512, 2048, torch.float32),
    (100, 1024, 8192, torch.float32), (128, 2048, 5120, torch.bfloat16), (7, 264, 1856, torch.float32)])
def test_gemm_small_m_split_k(fmt, M, N, K, dtype):
    """Small-M (decode) shapes take the split-K path: fp32 partials per K slice, reduced in a
    fixed split order inside the GEMM kernel -- deterministic, within the fp32 tolerance."""
    from paper_2509_23202_b200 import _lib
    assert _lib.lib().mrfp4_gemm_workspace(M, N, K, 0 if fmt == "mxfp4" else 1) > 0 or N >= 256 * 74
    rng = np.random.default_rng(M * 17 + N + K)
    A, W = random_container(rng, M, K, fmt), random_container(rng, N, K, fmt)
    y = run_gemm(A, W, dtype).float().cpu().numpy()
    ref = ref64(A, W)
    assert rel_fro(y, ref) <= (1e-5 if dtype == torch.float32 else 3e-3), rel_fro(y, ref)
    y2 = run_gemm(A, W, dtype).float().cpu().numpy()
    assert np.array_equal(y, y2)   # deterministic reduction order


def test_gemm_split_k_counters_rearm_across_shapes():
    """The in-kernel split-K reduction leaves its per-tile counters zero: shapes with different
    tile / split counts, interleaved on one stream (one shared workspace), keep their results."""
    rng = np.random.default_rng(11)
    cases = [(16, 4096, 4096, "nvfp4"), (3, 768, 2048, "mxfp4"), (64, 1024, 8192, "nvfp4")]
    data = [(random_container(rng, M, K, f), random_container(rng, N, K, f)) for M, N, K, f in cases]
    first = [run_gemm(A, W).cpu().numpy() for A, W in data]
    for _ in range(3):
        for (A, W), y0 in zip(reversed(data), reversed(first)):
            assert np.array_equal(run_gemm(A, W).cpu().numpy(), y0)
    for (A, W), y0 in zip(data, first):
        assert rel_fro(y0, ref64(A, W)) <= 1e-5


@pytest.mark.parametrize("fmt", ["mxfp4", "nvfp4"])
@pytest.mark.parametrize("M,N,K", [(512, 2048, 4096), (768, 2048, 5120), (300, 1280, 7168), (512, 9728, 4096)])
def test_gemm_2cta_bf16_shapes(fmt, M, N, K):
    """2-CTA kernel, bf16 output: ragged M, few tiles, one full wave plus a partial one."""
    rng = np.random.default_rng(M + N + K)
    A, W = random_container(rng, M, K, fmt), random_container(rng, N, K, fmt)
    y = run_gemm(A, W, torch.bfloat16).float().cpu().numpy()
    assert rel_fro(y, ref64(A, W)) <= 3e-3
    assert np.array_equal(y, run_gemm(A, W, torch.bfloat16).float().cpu().numpy())


@pytest.mark.parametrize("fmt", ["mxfp4", "nvfp4"])
def test_gemm_bf16_output_within_one_ulp(fmt):
    rng = np.random.default_rng(5)
    A, W = random_container(rng, 256, 1024, fmt), random_container(rng, 512, 1024, fmt)
    y = run_gemm(A, W, torch.bfloat16).float().cpu().numpy()
    ref = ref64(A, W)
    refb = torch.from_numpy(ref.astype(np.float32)).bfloat16().float().numpy()
    ulp = np.abs(refb) * 2.0 ** -7 + 1e-30
    assert (np.abs(y - refb) <= ulp * 1.01).mean() >= 0.999
    assert rel_fro(y, ref) <= 3e-3


@pytest.mark.parametrize("fmt", ["mxfp4", "nvfp4"])
def test_gemm_known_answer_single_group(fmt):
    """One nonzero group per row: every code x every scale code passes through exactly."""
    G = 32 if fmt == "mxfp4" else 16
    K = 256
    rng = np.random.default_rng(9)
    A = random_container(rng, 128, K, fmt, ts=1.0)
    W = random_container(rng, 256, K, fmt, ts=1.0)
    A.element_codes[:] = 0
    A.element_codes[:, :G] = np.arange(16, dtype=np.uint8)[np.arange(128 * G) % 16].reshape(128, G)
    A.scale_codes[:, 0] = (np.arange(128) % 100 + (20 if fmt == "mxfp4" else 1)).astype(np.uint8)
    y = run_gemm(A, W).cpu().numpy()
    np.testing.assert_allclose(y, ref64(A, W), rtol=1e-6, atol=1e-30)


@pytest.mark.parametrize("fmt", ["mxfp4", "nvfp4"])
@pytest.mark.parametrize("k", [0, 16, 32, 128])
def test_golden_linear(golden, fmt, k):
    """End to end through quantized_linear on the reference's own linear fixtures."""
    key = f"lin_{fmt}_k{k}"
    A = torch.from_numpy(golden[key + "_a"]).cuda().bfloat16()
    Wq = O.quantize_rtn(golden[key + "_w"], fmt, hadamard=k or None)
    t = P.MfpTensor(SPEC[fmt], Wq.rows, Wq.cols, Wq.codes.reshape(-1), Wq.scale_codes.reshape(-1),
                    Wq.tensor_scale, P.TransformSpec.hadamard(k) if k else None, None)
    w = P.prepare_weight(t)
    y = P.quantized_linear(A, w, out_dtype=torch.float32).cpu().numpy()
    ref = golden[key + "_y"]
    assert rel_fro(y, ref) <= 1e-5


@pytest.mark.parametrize("fmt", ["mxfp4", "nvfp4"])
def test_quantize_weight_matches_prepare_weight(fmt):
    rng = np.random.default_rng(2)
    W = O.bf16_round(rng.standard_normal((256, 512)) / 16)
    X = O.bf16_round(rng.standard_normal((64, 512)))
    tr = P.TransformSpec.hadamard(32)
    w_gpu = P.quantize_weight(torch.from_numpy(W).cuda().bfloat16(), SPEC[fmt], tr)
    Wq = O.quantize_rtn(W, fmt, hadamard=32)
    Aq = O.quantize_rtn(X, fmt, hadamard=32)
    y = P.quantized_linear(torch.from_numpy(X).cuda().bfloat16(), w_gpu, out_dtype=torch.float32)
    ref = O.linear_reference(Aq, Wq)
    assert rel_fro(y.cpu().numpy(), ref) <= 1e-4


def test_weight_validation():
    rng = np.random.default_rng(0)
    q = random_container(rng, 128, 256, "mxfp4")
    t = to_mfp(q)
    bad = P.MfpTensor(t.spec, t.rows, t.cols, t.codes, t.scale_codes, t.tensor_scale, None, (0.1, -3.0))
    with pytest.raises(P.DataError, match="scale_fit"):
        P.prepare_weight(bad)
    q2 = random_container(rng, 128, 96, "mxfp4")
    with pytest.raises(P.DataError, match="multiple of 64"):
        P.prepare_weight(to_mfp(q2))


@pytest.mark.parametrize("fmt,k,M", [("mxfp4", 32, 2048), ("mxfp4", 128, 1000), ("nvfp4", 16, 700), ("mxfp4", 32, 100)])
def test_host_pipeline_matches_device_call(fmt, k, M):
    """quantized_linear_host (row chunks over three streams for MXFP4) == quantized_linear."""
    rng = np.random.default_rng(M + k)
    K, N = 2048, 768
    X = torch.from_numpy(O.bf16_round(rng.standard_normal((M, K)))).bfloat16()
    W = torch.from_numpy(O.bf16_round(rng.standard_normal((N, K)) / 45)).bfloat16().cuda()
    w = P.quantize_weight(W, SPEC[fmt], P.TransformSpec.hadamard(k))
    ref = P.quantized_linear(X.cuda(), w).cpu()
    for chunk in (None, 256, 384):
        y = P.quantized_linear_host(X.pin_memory(), w, chunk_rows=chunk)
        torch.cuda.synchronize()
        assert y.device.type == "cpu" and torch.equal(y, ref), chunk
    out = torch.empty((M, N), dtype=torch.float32).pin_memory()
    P.quantized_linear_host(X, w, out=out)
    torch.cuda.synchronize()
    assert torch.equal(out, P.quantized_linear(X.cuda(), w, out_dtype=torch.float32).cpu())


@pytest.mark.parametrize("fmt", ["mxfp4", "nvfp4"])
@pytest.mark.parametrize("M,N,K", [(2048, 4096, 2048), (300, 640, 1024), (129, 1152, 512)])
@pytest.mark.parametrize("next_k", [0, 16, 32])
def test_requant_epilogue_matches_act_quant(fmt, M, N, K, next_k):
    """K2 with the next layer's MXFP4 act-quant in its epilogue == quantize_rtn of the bf16
    output, byte for byte (codes, swizzled scales incl. zero padding rows, tensor scale)."""
    rng = np.random.default_rng(M + N + next_k)
    X = torch.from_numpy(O.bf16_round(rng.standard_normal((M, K)))).cuda().bfloat16()
    W = torch.from_numpy(O.bf16_round(rng.standard_normal((N, K)) / np.sqrt(K))).cuda().bfloat16()
    w = P.quantize_weight(W, SPEC[fmt], P.TransformSpec.hadamard(16))
    tr = P.TransformSpec.hadamard(next_k) if next_k else None
    q, y = P.quantized_linear_requant(X, w, tr, keep_output=True, check=True)
    y_ref = P.quantized_linear(X, w)
    assert torch.equal(y, y_ref)
    ref = P.quantize_rtn(y_ref, SPEC["mxfp4"], transform=tr)
    assert torch.equal(q.codes, ref.codes) and torch.equal(q.sf, ref.sf)
    assert q.tensor_scale == ref.tensor_scale
    q2 = P.quantized_linear_requant(X, w, tr)          # without storing y
    assert torch.equal(q2.codes, ref.codes) and torch.equal(q2.sf, ref.sf)


def test_requant_rejects_unsupported():
    rng = np.random.default_rng(1)
    X = torch.from_numpy(O.bf16_round(rng.standard_normal((64, 512)))).cuda().bfloat16()   # M <= 128
    W = torch.from_numpy(O.bf16_round(rng.standard_normal((256, 512)) / 23)).cuda().bfloat16()
    w = P.quantize_weight(W, SPEC["mxfp4"], P.TransformSpec.hadamard(32))
    with pytest.raises(P.DataError):
        P.quantized_linear_requant(X, w)
    X2 = torch.from_numpy(O.bf16_round(rng.standard_normal((256, 512)))).cuda().bfloat16()
    with pytest.raises(P.DataError, match="static"):   # whole-y NVFP4 s_T cannot be fused
        P.quantized_linear_requant(X2, w, next_spec=SPEC["nvfp4"])
    with pytest.raises(P.DataError):
        P.quantized_linear_requant(X2, w, next_tensor_scale=1.0)   # MXFP4 has no global scale


@pytest.mark.parametrize("next_fmt,next_k", [("mxfp4", 64), ("mxfp4", 128), ("nvfp4", 0), ("nvfp4", 16),
                                             ("nvfp4", 64), ("nvfp4", 128)])
@pytest.mark.parametrize("M,N,K", [(256, 1024, 2048), (300, 2048, 1024)])
def test_requant_epilogue_all_blocks_and_nvfp4_static(next_fmt, next_k, M, N, K):
    """Next-layer requant with H64 / H128 (cross-segment stages inside the epilogue thread) and
    NVFP4 against a static global scale: byte-identical to K1 on the bf16 output, and to the
    oracle (quantize_rtn with that s_global) at the north-star bar."""
    rng = np.random.default_rng(M + N + next_k)
    X = torch.from_numpy(O.bf16_round(rng.standard_normal((M, K)))).cuda().bfloat16()
    W = torch.from_numpy(O.bf16_round(rng.standard_normal((N, K)) / np.sqrt(K))).cuda().bfloat16()
    w = P.quantize_weight(W, SPEC["mxfp4"], P.TransformSpec.hadamard(32))
    tr = P.TransformSpec.hadamard(next_k) if next_k else None
    y_ref = P.quantized_linear(X, w)
    st = None
    if next_fmt == "nvfp4":   # e.g. calibrated offline: 0.8 x this batch's dynamic s_T (some groups saturate)
        st = float(np.float32(P.quantize_rtn(y_ref, SPEC["nvfp4"], transform=tr).tensor_scale * 0.8))
    q, y = P.quantized_linear_requant(X, w, tr, next_spec=SPEC[next_fmt], next_tensor_scale=st, keep_output=True,
                                      check=True)
    assert torch.equal(y, y_ref)
    ref = P.quantize_rtn(y_ref, SPEC[next_fmt], transform=tr, static_tensor_scale=st)
    assert torch.equal(q.codes, ref.codes) and torch.equal(q.sf, ref.sf)
    assert q.tensor_scale == ref.tensor_scale
    ora = O.quantize_rtn(y_ref.float().cpu().numpy().astype(np.float64), next_fmt, hadamard=next_k or None,
                         static_ts=st)
    ec = O.unpack_nibbles(q.codes.cpu().numpy(), M * N).reshape(M, N)
    assert (ec == ora.element_codes).mean() >= 0.9999
    assert (q.scale_codes().cpu().numpy() == ora.scale_codes).mean() >= 0.9999


@pytest.mark.parametrize("fmt,k,M", [("nvfp4", 16, 16), ("mxfp4", 32, 16), ("nvfp4", 128, 256), ("mxfp4", 32, 512)])
def test_graphed_linear_matches_eager(fmt, k, M):
    """The CUDA-graph replay of K1 + K2 (+ split-K reduce) equals the eager call, call after call."""
    rng = np.random.default_rng(M + k)
    K, N = 4096, 1024
    W = torch.from_numpy(O.bf16_round(rng.standard_normal((N, K)) / 64)).cuda().bfloat16()
    w = P.quantize_weight(W, SPEC[fmt], P.TransformSpec.hadamard(k))
    g = P.GraphedLinear(w, M)
    for seed in range(3):
        X = torch.from_numpy(O.bf16_round(np.random.default_rng(seed).standard_normal((M, K)))).cuda().bfloat16()
        y = g(X).clone()
        torch.cuda.synchronize()
        assert torch.equal(y, P.quantized_linear(X, w))


@pytest.mark.parametrize("fmt,M", [("mxfp4", 512), ("nvfp4", 300)])
def test_fused_gather_peer_stores_emulated(fmt, M):
    """The all-gather fused into K2's epilogue (mrfp4_gemm_peers), emulated on one GPU: 4 ranks'
    output buffers are local tensors; each rank's shard GEMM stores its column block into all
    four.  Every buffer must equal the unsharded linear, bit for bit."""
    from paper_2509_23202_b200.quantize import act_quant_into, alloc_result
    from paper_2509_23202_b200.sharded import gemm_into_peers
    P_, K, N = 4, 1024, 2048
    rng = np.random.default_rng(M)
    X = torch.from_numpy(O.bf16_round(rng.standard_normal((M, K)))).cuda().bfloat16()
    W = torch.from_numpy(O.bf16_round(rng.standard_normal((N, K)) / 32)).cuda().bfloat16()
    k = 32 if fmt == "mxfp4" else 16
    w = P.quantize_weight(W, SPEC[fmt], P.TransformSpec.hadamard(k))
    ref = P.quantized_linear(X, w)
    a = alloc_result(M, K, w.fmt, k, "cuda")
    act_quant_into(X, w.fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    bufs = [torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(P_)]
    n = N // P_
    for r in range(P_):
        gemm_into_peers(a, w.shard(r, P_), [b[:, r * n:(r + 1) * n] for b in bufs])
    torch.cuda.synchronize()
    for b in bufs:
        assert torch.equal(b, ref)
