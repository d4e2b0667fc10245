"""Per-stage MMA-issuer timeline (clock64) of cluster 0 for the first 4 tiles of the 2-CTA GEMM."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
L = _lib.lib()
L.mrfp4_debug_gemm_timestamps.argtypes = [ctypes.c_void_p]
M, K, N = [int(v) for v in sys.argv[1:4]]
fmt = int(sys.argv[4]) if len(sys.argv) > 4 else 0
spec = P.FormatSpec.mxfp4() if fmt == 0 else P.FormatSpec.nvfp4()
x = torch.randn(M, K, device="cuda").bfloat16()
w = P.quantize_weight((torch.randn(N, K, device="cuda") / K**0.5).bfloat16(), spec, None)
a = alloc_result(M, K, w.fmt, 0, "cuda")
act_quant_into(x, w.fmt, 0, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    P.gemm(a, w, out)
buf = torch.zeros(2048, dtype=torch.int64, device="cuda")
L.mrfp4_debug_gemm_timestamps(buf.data_ptr())
P.gemm(a, w, out)
torch.cuda.synchronize()
L.mrfp4_debug_gemm_timestamps(None)
t = buf.cpu().tolist()
nkb = (K + 511) // 512
for tl in range(4):
    b = tl * 260
    if t[b] == 0:
        break
    full = [t[b + 2 + 2 * k] for k in range(min(nkb, 128))]
    done = [t[b + 3 + 2 * k] for k in range(min(nkb, 128))]
    gaps = [full[k + 1] - full[k] for k in range(len(full) - 1)]
    issue = [done[k] - full[k] for k in range(len(full))]
    print(f"tile {tl}: start {t[b] - t[0]}, tempty wait {t[b + 1] - t[b]}, first full {full[0] - t[b + 1]}, "
          f"stage period mean {sum(gaps) / max(len(gaps), 1):.0f} (min {min(gaps) if gaps else 0}, max {max(gaps) if gaps else 0}), "
          f"issue mean {sum(issue) / len(issue):.0f}, tile end {done[-1] - t[0]}")
    print("   periods:", gaps[:24])
