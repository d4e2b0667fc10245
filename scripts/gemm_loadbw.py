"""Load-pipeline-only GEMM (debug mode 64: no MMAs) at several grid sizes: per-SM vs chip-level limit."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
L = _lib.lib()
for f in ("mrfp4_debug_gemm_mode", "mrfp4_debug_gemm_kernel", "mrfp4_debug_gemm_grid"):
    getattr(L, f).argtypes = [ctypes.c_int]
L.mrfp4_debug_gemm_kernel(2)
M = K = N = 8192
x = torch.randn(M, K, device="cuda").bfloat16()
w = P.quantize_weight((torch.randn(N, K, device="cuda") / K**0.5).bfloat16(), P.FormatSpec.mxfp4(), None)
a = alloc_result(M, K, w.fmt, 0, "cuda")
act_quant_into(x, w.fmt, 0, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
mode = int(os.environ.get("MODE", "64"))
L.mrfp4_debug_gemm_mode(mode)
for grid in (148, 112, 74, 38, 16):
    L.mrfp4_debug_gemm_grid(grid)
    for _ in range(2):
        P.gemm(a, w, out)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        P.gemm(a, w, out)
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / 5 * 1e-3
    tiles = (M // 256) * (N // 256)
    byts = tiles * (K // 256) * 2 * 128 * 128 * 2  # A + B per tile-kb, both CTAs
    print(json.dumps(dict(mode=mode, grid=grid, us=round(t * 1e6, 1), chip_GBs=round(byts / t / 1e9),
                          per_sm_GBs=round(byts / t / 1e9 / grid, 1))))
L.mrfp4_debug_gemm_grid(0); L.mrfp4_debug_gemm_mode(0)
