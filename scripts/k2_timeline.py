"""Where the 2-CTA GEMM's MMA thread waits (MRFP4_TRACE build, cluster 0): per tile the wait for
the epilogue to free the accumulator (tempty), per stage the waits for the SF slot (sf_full) and
the A/B stage (full), and the issue time in between.
Usage: MRFP4_LIB=build/trace/libmrfp4.so python scripts/k2_timeline.py [config]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import act_quant_into, alloc_result

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2-up-nv"
name, M, K, N, fmt, had = bench.CONFIGS[cfg]
L = _lib.lib()
L.mrfp4_debug_gemm_timestamps.argtypes = [ctypes.c_void_p]
L.mrfp4_debug_gemm_mode.argtypes = [ctypes.c_int]
L.mrfp4_debug_gemm_mode(int(os.environ.get("MODE", "0")))   # 2: load pipeline only (no cp / MMA)
spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
x = torch.randn(M, K, device="cuda").bfloat16()
w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16(), spec, P.TransformSpec.hadamard(had))
a = alloc_result(M, K, w.fmt, had, "cuda")
act_quant_into(x, w.fmt, had, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
buf = torch.zeros(2 * 8192, dtype=torch.int64, device="cuda")
for _ in range(3):
    P.gemm(a, w, y)
flush.zero_()
L.mrfp4_debug_gemm_timestamps(buf.data_ptr())
P.gemm(a, w, y)
torch.cuda.synchronize()
L.mrfp4_debug_gemm_timestamps(None)
t = buf.view(-1, 2).cpu().numpy()
t = t[t[:, 0] != 0]
clk, tag = t[:, 0].astype(np.int64), t[:, 1]
d = np.diff(clk)
names = {1: "tempty wait (epilogue drain)", 2: "sf_full wait", 3: "full (A/B) wait", 4: "cp + MMA issue", 0: "tile switch"}
acc = {v: 0 for v in names.values()}
for i in range(len(d)):
    acc[names[int(tag[i + 1])]] += int(d[i])
stages = int((tag == 3).sum())
tiles = int((tag == 0).sum())
total = int(clk[-1] - clk[0])
ideal = stages * 8 * 128
print(f"{cfg}: cluster 0 ran {tiles} tiles, {stages} stages, {total} cycles; ideal MMA {ideal} ({ideal / total:.1%})")
for k, v in acc.items():
    print(f"  {k:32s} {v:9d} cycles {v / total:6.1%}")
per_stage = np.diff(clk[tag == 3])
print("  stage-to-stage cycles: median %d p90 %d max %d" % (np.median(per_stage), np.percentile(per_stage, 90), per_stage.max()))
