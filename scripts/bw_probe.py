"""Reference floors: torch read-reduce and copy kernels on the K1 input sizes (CUDA events, L2 flushed)."""
import sys, os, json
import torch
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")

def timeit(fn, iters=30, warm=5):
    for _ in range(warm):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    torch.cuda.synchronize()
    for s, e in ev:
        flush.zero_()
        s.record(); fn(); e.record()
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) for s, e in ev)
    return ts[len(ts) // 2] * 1e-3

for M, K in [(16, 4096), (2048, 8192), (2048, 14336), (2048, 28672), (8192, 28672)]:
    x = torch.randn(M, K, device="cuda").bfloat16()
    y = torch.empty_like(x)
    q = torch.empty(M, K // 4, dtype=torch.int32, device="cuda")
    t_sum = timeit(lambda: torch.sum(x, dim=1))
    t_copy = timeit(lambda: y.copy_(x))
    t_empty = timeit(lambda: torch.cuda._sleep(0))
    nb = M * K * 2
    print(json.dumps(dict(M=M, K=K, sum_us=round(t_sum * 1e6, 2), sum_gbs=round(nb / t_sum / 1e9),
                          copy_us=round(t_copy * 1e6, 2), copy_gbs=round(2 * nb / t_copy / 1e9),
                          sleep0_us=round(t_empty * 1e6, 2))))
