"""NVFP4 K1 phase timeline (globaltimer): phase-1 end, barrier release, phase-2 end per warp."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
L = _lib.lib()
L.mrfp4_debug_k1_trace.argtypes = [ctypes.c_void_p]
M, K, k = [int(v) for v in sys.argv[1:4]]
x = torch.randn(M, K, device="cuda").bfloat16()
a = alloc_result(M, K, 1, k, "cuda")
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    act_quant_into(x, 1, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
buf = torch.zeros(8 * 148 * 24, dtype=torch.int64, device="cuda")
L.mrfp4_debug_k1_trace(buf.data_ptr())
if not os.environ.get("WARM"): flush.zero_(); flush.sum(dtype=torch.int32)
act_quant_into(x, 1, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
torch.cuda.synchronize()
L.mrfp4_debug_k1_trace(None)
t = buf.view(-1, 8).cpu()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min().item()
f = lambda v: [round(float(torch.quantile((v - t0).double(), z)) / 1000, 2) for z in (0, .5, .9, 1)]
print("start", f(t[:, 0]), "| phase-1 end", f(t[:, 3]), "| barrier release", f(t[:, 4]), "| phase-2 end", f(t[:, 1]))
# clock-skew check: per CTA, barrier release - latest phase-1 end of any warp in the grid
nw = int(os.environ.get("WARPS", "24"))
cta = torch.arange(len(t)) // nw
p1max = t[:, 3].max()
rel = t[:, 4]
print("release - global max phase-1 end (us) q0/50/100:", [round(float(torch.quantile((rel - p1max).double(), z)) / 1000, 2) for z in (0, .5, 1)])
# per CTA: latest phase-1 end, release (us from start)
for c in range(int(cta.max()) + 1):
    m = cta == c
    print("cta", c, "p1 end max", round((t[m, 3].max() - t0).item() / 1000, 2), "release", round((t[m, 4].min() - t0).item() / 1000, 2),
          "sm", int(t[m, 2][0].item() >> 32), "n", int((t[m, 2] & 0xffffffff).sum().item()))
