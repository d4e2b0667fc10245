"""K1 time vs the practical per-size floor: torch read-only sweep and D2D copy of X, L2 flushed."""
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
shapes = [(2048, 14336, 0, 32), (2048, 14336, 1, 16), (2048, 8192, 1, 16), (2048, 8192, 0, 32), (2048, 28672, 1, 16),
          (2048, 5120, 1, 128), (2048, 5120, 0, 128), (16, 4096, 1, 16), (8192, 28672, 0, 32), (8192, 8192, 1, 16)]
for M, K, fmt, k in shapes:
    x = torch.randn(M, K, device="cuda").bfloat16()
    a = alloc_result(M, K, fmt, k, "cuda")
    y = torch.empty_like(x)
    o = torch.empty(M * K // 8, dtype=torch.int32, device="cuda")
    t1 = timeit(lambda: act_quant_into(x, fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch))
    tr = timeit(lambda: torch.amax(x.view(torch.int32), dim=1))
    tc = timeit(lambda: y.copy_(x))
    G = 32 if fmt == 0 else 16
    by = M * K * (2.5 + 1 / G)
    print(json.dumps(dict(M=M, K=K, fmt=fmt, k=k, k1_us=round(t1, 2), k1_gbs=round(by / t1 / 1e3), read_us=round(tr, 2),
                          read_gbs=round(M * K * 2 / tr / 1e3), copy_us=round(tc, 2), copy_gbs=round(M * K * 4 / tc / 1e3))))
