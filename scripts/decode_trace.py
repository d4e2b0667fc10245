"""Per-CTA timeline of the fused decode kernel (globaltimer, us from the first CTA start).
Needs a trace build: VSRC=linear_decode scripts/build_variant.sh trace_dec -DMRFP4_TRACE, then
MRFP4_LIB=build/var_trace_dec/libmrfp4.so python scripts/decode_trace.py M K N fmt(0 mx/1 nv) k [noflush]."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.linear import _linear_decode, decode_workspace_bytes
L = _lib.lib()
fn = L.mrfp4_debug_decode_trace
fn.argtypes = [ctypes.c_void_p]
M, K, N, fmt, k = [int(v) for v in sys.argv[1:6]]
spec = P.FormatSpec.mxfp4() if fmt == 0 else P.FormatSpec.nvfp4()
w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16(), spec, P.TransformSpec.hadamard(k))
x = torch.randn(M, K, device="cuda").bfloat16()
y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
ws = torch.zeros(max(decode_workspace_bytes(M, w), 1), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    _linear_decode(x, w, y, ws, None)
buf = torch.zeros(16 * 2048, dtype=torch.int64, device="cuda")
st = L.mrfp4_debug_stamp
st.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
stamps = torch.zeros(4, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
fn(buf.data_ptr())
if "noflush" not in sys.argv:
    flush.zero_()
    flush.sum(dtype=torch.int32)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
st(stamps.data_ptr(), sp)
_linear_decode(x, w, y, ws, None)
st(stamps.data_ptr() + 8, sp)
e1.record()
torch.cuda.synchronize()
fn(None)
print(f"events around stamp+decode+stamp: {e0.elapsed_time(e1) * 1e3:.2f} us")
t = buf.view(-1, 16).cpu()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min().item()
q = lambda c: [round(float(torch.quantile((t[:, c] - t0).double(), z)) / 1000, 2) for z in (0, .5, .9, 1)]
print(f"M={M} K={K} N={N} fmt={fmt}: CTAs {len(t)}")
s_ = stamps.cpu()
print(f"  stamp kernel before -> first CTA start: {(t0 - s_[0].item()) / 1000:.2f} us; "
      f"last CTA stored -> stamp kernel after: {(s_[1].item() - t[:, 5].max().item()) / 1000:.2f} us")
for name, c in (("start", 0), ("after pdl_wait", 1), ("X loaded+rotated", 6), ("cluster wait done", 8), ("CTA max pushed", 7), ("max landed", 12), ("consts done", 13), ("global max done", 2), ("X quantized", 3), ("MMAs done", 4), ("partial in regs", 9), ("partial pushed", 10), ("partials landed", 11), ("stored", 5)):
    if fmt == 0 and c in (7, 12, 13):
        continue
    print(f"  {name:18s} q0/50/90/100 us: {q(c)}")
