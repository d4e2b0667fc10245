"""Per-k-block timestamps of the MMA thread (CTA 0, first tile) in the 1-CTA GEMM."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
L = _lib.lib()
for f in ("mrfp4_debug_gemm_mode", "mrfp4_debug_gemm_kernel"):
    getattr(L, f).argtypes = [ctypes.c_int]
L.mrfp4_debug_gemm_timestamps.argtypes = [ctypes.c_void_p]
buf = torch.zeros(128, dtype=torch.int64, device="cuda")
L.mrfp4_debug_gemm_timestamps(buf.data_ptr())
L.mrfp4_debug_gemm_kernel(int(os.environ.get('KERNEL', '1')))
M, K, N = 2048, 14336, 4096
x = torch.randn(M, K, device="cuda").bfloat16()
w = P.quantize_weight((torch.randn(N, K, device="cuda") / K**0.5).bfloat16(), P.FormatSpec.mxfp4(), None)
a = alloc_result(M, K, w.fmt, 0, "cuda")
act_quant_into(x, w.fmt, 0, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
L.mrfp4_debug_gemm_grid.argtypes = [ctypes.c_int]
for grid, mode in ((0, 0), (0, 3), (0, 5), (0, 6), (2, 5)):
    L.mrfp4_debug_gemm_grid(grid)
    L.mrfp4_debug_gemm_mode(mode)
    for _ in range(3):
        P.gemm(a, w, out)
    torch.cuda.synchronize()
    t = buf.cpu().tolist()
    starts = t[0::2][:56]; waits = [t[2*i+1] - t[2*i] for i in range(56)]
    d = [starts[i+1] - starts[i] for i in range(55)]
    print(f"grid {grid} mode {mode}: per-kb cycles {d[:12]} ... median {sorted(d)[len(d)//2]}; full-wait cycles {waits[:12]} median {sorted(waits)[28]}")
