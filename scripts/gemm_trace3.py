"""Per-k-block MMA issue timeline (globaltimer ns) of clusters 0/37/73, first 2 tiles, 2-CTA GEMM on C1."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
L = _lib.lib()
L.mrfp4_debug_gemm_kernel.argtypes = [ctypes.c_int]
L.mrfp4_debug_gemm_timestamps.argtypes = [ctypes.c_void_p]
L.mrfp4_debug_gemm_mode.argtypes = [ctypes.c_int]
L.mrfp4_debug_gemm_mode(int(os.environ.get("MODE", "0")))
M, K, N = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (2048, 14336, 4096))]
x = torch.randn(M, K, device="cuda").bfloat16()
w = P.quantize_weight((torch.randn(N, K, device="cuda") / K**0.5).bfloat16(), P.FormatSpec.mxfp4(), None)
a = alloc_result(M, K, w.fmt, 0, "cuda")
act_quant_into(x, w.fmt, 0, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    P.gemm(a, w, out)
buf = torch.zeros(8192, dtype=torch.int64, device="cuda")
L.mrfp4_debug_gemm_timestamps(buf.data_ptr())
flush.zero_(); torch.cuda.synchronize()
P.gemm(a, w, out)
torch.cuda.synchronize()
L.mrfp4_debug_gemm_timestamps(None)
t = buf.cpu().tolist()
w = [(t[1800 + 2 * k], t[1801 + 2 * k]) for k in range(56)]
waits = [b - a for a, b in w if a]
iters = [w[k + 1][0] - w[k][0] for k in range(55) if w[k][0] and w[k + 1][0]]
print("cluster 0 tile 1: full-wait cycles per kb:", waits[4:20], "iter cycles:", iters[4:20])
print("mean wait", sum(waits) / max(len(waits), 1), "mean iter", sum(iters) / max(len(iters), 1))
n = t[422]
for i in range(min(n, 4)):
    print(f"tile {i}: start clk {t[400+4*i]-t[400]}, tempty wait {t[402+4*i]-t[400+4*i]}, mainloop {t[403+4*i]-t[402+4*i]}")
seg = []
for k in range(4, 20):
    a0, a1, w0, w1, c = t[2000 + 4 * k], t[2001 + 4 * k], t[1800 + 2 * k], t[1801 + 2 * k], t[2000 + 4 * (k + 1)]
    seg.append((w0 - a0, w1 - w0, a1 - w1, c - a1))
print("per kb: [issue3, wait, issue1, commit+loop->next]:", seg[:10])
