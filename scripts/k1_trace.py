"""Per-warp K1 timeline (globaltimer ns): launch ramp, first-segment latency, tail."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
L = _lib.lib()
L.mrfp4_debug_k1_trace.argtypes = [ctypes.c_void_p]
M, K, fmt, k = [int(v) for v in sys.argv[1:5]]
x = torch.randn(M, K, device="cuda").bfloat16()
a = alloc_result(M, K, fmt, k, "cuda")
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    act_quant_into(x, fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
buf = torch.zeros(8 * 148 * 24, dtype=torch.int64, device="cuda")
L.mrfp4_debug_k1_trace(buf.data_ptr())
flush.zero_(); flush.sum(dtype=torch.int32)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
act_quant_into(x, fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
e.record()
torch.cuda.synchronize()
L.mrfp4_debug_k1_trace(None)
t = buf.view(-1, 8).cpu()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min().item()
st, end = (t[:, 0] - t0).float(), (t[:, 1] - t0).float()
first = st
n = (t[:, 2] & 0xFFFFFFFF)
q = lambda v: [round(float(torch.quantile(v, z)) / 1000, 2) for z in (0.0, 0.5, 0.9, 1.0)]
print(f"event {s.elapsed_time(e) * 1000:.2f} us, warps {len(t)}, items/warp {n.min().item()}..{n.max().item()}")
print("start   us q0/50/90/100:", q(st))
print("end     us:", q(end))
if (t[:, 3] > 0).any():
    print("NVFP4 phase-1 end us:", q((t[:, 3] - t0).float()), " barrier released us:", q((t[:, 4] - t0).float()))
sm = (t[:, 2] >> 32)
persm = torch.zeros(int(sm.max()) + 1)
persm.index_reduce_(0, sm, end, "amax", include_self=False)
print("per-SM last end us q0/10/50/90/100:", [round(float(torch.quantile(persm, z)) / 1000, 2) for z in (0, .1, .5, .9, 1)])
fs = torch.zeros(int(sm.max()) + 1)
fs.index_reduce_(0, sm, first, "mean", include_self=False)
print("per-SM mean first us q0/10/50/90/100:", [round(float(torch.quantile(fs, z)) / 1000, 2) for z in (0, .1, .5, .9, 1)])
me = torch.zeros(int(sm.max()) + 1)
me.index_reduce_(0, sm, end, "mean", include_self=False)
print("per-SM mean end us q0/10/50/90/100:", [round(float(torch.quantile(me, z)) / 1000, 2) for z in (0, .1, .5, .9, 1)])
cta = torch.arange(len(t)) // int(os.environ.get('WARPS', '24'))
cmax = torch.zeros(int(cta.max()) + 1); cmax.index_reduce_(0, cta, end, "amax", include_self=False)
cmean = torch.zeros(int(cta.max()) + 1); cmean.index_reduce_(0, cta, end, "mean", include_self=False)
print("per-CTA max end q0/50/100:", [round(float(torch.quantile(cmax, z)) / 1000, 2) for z in (0, .5, 1)],
      " per-CTA mean end q0/50/100:", [round(float(torch.quantile(cmean, z)) / 1000, 2) for z in (0, .5, 1)])
print("corr(SM mean first, SM last end):", round(float(torch.corrcoef(torch.stack([fs, persm]))[0, 1]), 3))
for v in sorted(set(n.tolist()))[:12]:
    sel = n == v
    print(f"  warps with {v} items: {int(sel.sum())}, end median {float(end[sel].median()) / 1000:.2f} us")
