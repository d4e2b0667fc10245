"""Step time: L2 flush before each step (per-step events) vs rotating input sets > L2 (back to back)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
cfgs = {"c1": (2048, 14336, 4096, "mxfp4", 32), "c2-up-nv": (2048, 8192, 28672, "nvfp4", 16),
        "c2-down-mx": (2048, 28672, 8192, "mxfp4", 32), "c3-gateup": (2048, 5120, 51200, "nvfp4", 128)}
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
fr = torch.ones(64 * 2**20, dtype=torch.int32, device="cuda")
for name in sys.argv[1:] or ["c1"]:
    M, K, N, fmt, had = cfgs[name]
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    tr = P.TransformSpec.hadamard(had)
    per_set = M * K * 2 + N * K * 0.5625 + M * N * 2 + M * K * 0.5625
    R = max(2, int(-(-3 * 126e6 // per_set)))
    sets = []
    for r in range(R):
        x = torch.randn(M, K, device="cuda").bfloat16()
        w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** .5).bfloat16(), spec, tr)
        a = alloc_result(M, K, w.fmt, had, "cuda")
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        sets.append((x, w, a, y))
    def step(i):
        x, w, a, y = sets[i % R]
        act_quant_into(x, w.fmt, had, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
        P.gemm(a, w, y)
    def k1(i):
        x, w, a, y = sets[i % R]
        act_quant_into(x, w.fmt, had, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    def k2(i):
        x, w, a, y = sets[i % R]
        P.gemm(a, w, y)
    def flushed(fn, n=50):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for i, (s, e) in enumerate(ev):
            flush.zero_(); fr.sum(dtype=torch.int32)
            s.record(); fn(i); e.record()
        torch.cuda.synchronize()
        return sum(s.elapsed_time(e) for s, e in ev) / n * 1e3
    def rotating(fn, n=200):
        for i in range(2 * R): fn(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for i in range(n): fn(i)
        e.record(); torch.cuda.synchronize()
        return s.elapsed_time(e) / n * 1e3
    for fn in (step, k1, k2): fn(0)
    out = dict(cfg=name, R=R, step_flush=flushed(step), step_rot=rotating(step), k1_flush=flushed(k1),
               k1_rot=rotating(k1), k2_flush=flushed(k2), k2_rot=rotating(k2))
    G = 32 if fmt == "mxfp4" else 16
    out["k1_rot_gbs"] = M * K * (2.5 + 1 / G) / out["k1_rot"] / 1e3
    out["k1_flush_gbs"] = M * K * (2.5 + 1 / G) / out["k1_flush"] / 1e3
    out["tflops_rot"] = 2 * M * N * K / out["step_rot"] / 1e6
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in out.items()}))
    del sets
    torch.cuda.empty_cache()
