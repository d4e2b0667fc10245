"""How much does the L2-flush method cost the next timed kernel? (sleep0 and a 58.7 MB copy)"""
import json
import torch
big = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
big2 = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
x = torch.randn(2048, 14336, device="cuda").bfloat16()
y = torch.empty_like(x)

def flush_write():
    big.zero_()

def flush_write_then_read():
    big.zero_()
    big2.sum(dtype=torch.int32)

def none():
    pass

def timeit(pre, fn, iters=30):
    for _ in range(5):
        pre(); fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    torch.cuda.synchronize()
    for s, e in ev:
        pre()
        s.record(); fn(); e.record()
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) for s, e in ev)
    return round(ts[len(ts) // 2] * 1e3, 2)

for name, pre in [("write", flush_write), ("write+read", flush_write_then_read), ("none", none)]:
    print(json.dumps(dict(flush=name, sleep0_us=timeit(pre, lambda: torch.cuda._sleep(0)),
                          copy_us=timeit(pre, lambda: y.copy_(x)))))
