"""Decode path vs K1 + K2 (forced in a subprocess via MRFP4_DECODE=0) on shapes the two-segment
cluster instantiation takes; flushed L2, CUDA events."""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = r"""
import sys, torch, json
sys.path.insert(0, sys.argv[1])
import paper_2509_23202_b200 as P
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
for (M, K, N) in ((16, 14336, 512), (24, 4096, 1024), (32, 4096, 1024), (32, 4096, 2048)):
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16(), P.FormatSpec.nvfp4(), P.TransformSpec.hadamard(16))
    x = torch.randn(M, K, device="cuda").bfloat16()
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    for _ in range(5): P.quantized_linear(x, w, out=y)
    ev = []
    for _ in range(100):
        flush.zero_(); flush.sum(dtype=torch.int32)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); P.quantized_linear(x, w, out=y); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    res[f"{M}x{K}->{N}"] = sum(p.elapsed_time(q) for p, q in ev) / len(ev) * 1e3
print(json.dumps(res))
"""
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {}
for d in ("1", "0"):
    r = subprocess.run([sys.executable, "-c", CODE, root], env=dict(os.environ, MRFP4_DECODE=d), capture_output=True, text=True)
    out[d] = json.loads(r.stdout.strip().splitlines()[-1])
for k in out["1"]:
    print(f"{k:18s} decode {out['1'][k]:6.1f} us   K1+K2 {out['0'][k]:6.1f} us")
