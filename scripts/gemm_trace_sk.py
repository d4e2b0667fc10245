"""Per-CTA timeline (globaltimer) of the 1-CTA split-K GEMM at a decode shape, after K1 (PDL):
0 start, 1 setup done, 2 producer past the PDL wait, 3 first stage landed, 4 accumulator ready,
5 partial stored, 6 all splits arrived, 7 slice reduced.  Quantiles over CTAs, us from first start."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
L = _lib.lib()
L.mrfp4_debug_gemm_timestamps.argtypes = [ctypes.c_void_p]
M, K, N = [int(v) for v in sys.argv[1:4]]
fmt, hk = (1, 16) if (len(sys.argv) < 5 or sys.argv[4] == "nvfp4") else (0, 32)
spec = P.FormatSpec.nvfp4() if fmt else P.FormatSpec.mxfp4()
x = torch.randn(M, K, device="cuda").bfloat16()
w = P.quantize_weight((torch.randn(N, K, device="cuda") / K**0.5).bfloat16(), spec, P.TransformSpec.hadamard(hk))
a = alloc_result(M, K, w.fmt, hk, "cuda")
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
step = lambda: (act_quant_into(x, w.fmt, hk, a.codes, a.sf, a.tensor_scale_dev, a.scratch), P.gemm(a, w, out))
for _ in range(5): step()
torch.cuda.synchronize()
buf = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
for warm in (False, True):
    buf.zero_()
    if not warm: flush.zero_(); flush.sum(dtype=torch.int32)
    L.mrfp4_debug_gemm_timestamps(buf.data_ptr())
    step()
    torch.cuda.synchronize()
    L.mrfp4_debug_gemm_timestamps(None)
    t = buf.view(-1, 8).cpu()
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min().item()
    names = ["start", "setup", "pdl", "stage0", "acc", "partial", "arrived", "reduced"]
    print("warm" if warm else "flushed", len(t), "CTAs")
    for i, n in enumerate(names):
        v = t[:, i]; v = v[v > 0]
        if len(v):
            print(f"  {n:8s}", [round(float(torch.quantile((v - t0).double(), z)) / 1000, 2) for z in (0, .5, .9, 1)])
