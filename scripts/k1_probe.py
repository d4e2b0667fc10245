"""K1 (act-quant) device time and GB/s for the bench configs (CUDA events, L2 flushed)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into

flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]

def timeit(fn, iters=100, warm=5):
    """Median device time; all iterations enqueued before one sync (the host runs ahead)."""
    for _ in range(warm):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    torch.cuda.synchronize()
    for s, e in ev:
        flush.zero_(); flush.sum(dtype=torch.int32)
        s.record(); fn(); e.record()
    torch.cuda.synchronize()
    ts = [s.elapsed_time(e) for s, e in ev]
    return sum(ts) / len(ts) * 1e-3  # mean: event times are quantized (~2 us steps)

for M, K, fmt, k in [(2048, 14336, 0, 32), (2048, 14336, 1, 16), (2048, 8192, 1, 16), (2048, 28672, 0, 32),
                     (2048, 28672, 1, 16), (8192, 28672, 0, 32), (2048, 5120, 1, 128), (2048, 25600, 1, 128),
                     (16, 4096, 1, 16), (8192, 8192, 1, 16)]:
    x = torch.randn(M, K, device="cuda").bfloat16()
    a = alloc_result(M, K, fmt, k, "cuda")
    t = timeit(lambda: act_quant_into(x, fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch))
    G = 32 if fmt == 0 else 16
    by = M * K * (2.5 + 1 / G)
    print(json.dumps(dict(M=M, K=K, fmt=["mxfp4", "nvfp4"][fmt], k=k, us=round(t * 1e6, 2),
                          gbs=round(by / t / 1e9), frac=round(by / t / 1e9 / peak, 3))))
