"""Interleaved A/B of K1 env-knob variants in one process (knobs are read per call).
usage: k1_ab.py 'NAME=V,NAME2=V2' 'NAME=V' ...   (each arg is one variant; '' = defaults)"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
def timeit(fn, iters=40):
    for _ in range(3): fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for s, e in ev:
        flush.zero_(); flush.sum(dtype=torch.int32)
        s.record(); fn(); e.record()
    torch.cuda.synchronize()
    return sum(s.elapsed_time(e) for s, e in ev) / iters * 1e3
variants = sys.argv[1:] or [""]
shapes = [(2048, 14336, 0, 32), (2048, 14336, 1, 16), (2048, 8192, 1, 16), (2048, 28672, 1, 16), (2048, 5120, 1, 128),
          (16, 4096, 1, 16), (8192, 28672, 0, 32), (8192, 8192, 1, 16)]
for M, K, fmt, k in shapes:
    x = torch.randn(M, K, device="cuda").bfloat16()
    a = alloc_result(M, K, fmt, k, "cuda")
    res = {v: [] for v in variants}
    for rep in range(3):
        for v in variants:
            keys = []
            for kv in filter(None, v.split(",")):
                n, val = kv.split("="); os.environ[n] = val; keys.append(n)
            res[v].append(timeit(lambda: act_quant_into(x, fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)))
            for n in keys: del os.environ[n]
    print(json.dumps(dict(M=M, K=K, fmt=fmt, k=k, **{v or "default": round(sum(t) / 3, 2) for v, t in res.items()})))
