import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
L = _lib.lib()
L.mrfp4_debug_gemm_kernel.argtypes = [ctypes.c_int]
L.mrfp4_debug_gemm_timestamps.argtypes = [ctypes.c_void_p]
buf = torch.zeros(512, dtype=torch.int64, device="cuda")
L.mrfp4_debug_gemm_timestamps(buf.data_ptr())
L.mrfp4_debug_gemm_kernel(2)
M, K, N = 2048, 14336, 4096
x = torch.randn(M, K, device="cuda").bfloat16()
w = P.quantize_weight((torch.randn(N, K, device="cuda") / K**0.5).bfloat16(), P.FormatSpec.mxfp4(), None)
a = alloc_result(M, K, w.fmt, 0, "cuda")
act_quant_into(x, w.fmt, 0, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    P.gemm(a, w, out)
torch.cuda.synchronize()
t = buf.cpu().tolist()
t0 = t[256]
for kb in range(0, 16):
    print(f"kb {kb:2d}: prod wait_empty@{t[256+2*kb]-t0:7d}..{t[257+2*kb]-t0:7d}  stager sf_full wait@{t[128+4*kb]-t0:7d}..{t[129+4*kb]-t0:7d}  mma full@{t[4*kb]-t0:7d}..{t[4*kb+1]-t0:7d} sf_ready..{t[4*kb+2]-t0:7d}")
for kb in range(8, 16):
    m = t[4*kb:4*kb+4]; st = t[128+4*kb:128+4*kb+4]
    print(f"kb {kb}: mma iter {t[4*(kb+1)]-m[0]:6d} wait_full {m[1]-m[0]:5d} wait_sf {m[2]-m[1]:5d} | stager iter {t[128+4*(kb+1)]-st[0]:6d} wait_sf_full {st[1]-st[0]:5d} lds+sttm {st[2]-st[1]:5d} wait_st {st[3]-st[2]:5d}")

n = t[422]
print("tiles", n)
for i in range(n):
    print(f"tile {i}: start clk {t[400+4*i]-t[400]}, tempty wait {t[402+4*i]-t[400+4*i]}, mainloop issue {t[403+4*i]-t[402+4*i]}")
print("total clk", t[420]-t[400], "ns", t[421]-t[401], "MHz", (t[420]-t[400])/(t[421]-t[401])*1e3)
