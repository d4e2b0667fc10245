"""Fixed cost of the event harness: empty-ish kernels vs K1 (c1), with and without PDL, flush before each."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
def timeit(fn, iters=200, fl=True):
    for _ in range(5): fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for s, e in ev:
        if fl:
            flush.zero_(); flush.sum(dtype=torch.int32)
        s.record(); fn(); e.record()
    torch.cuda.synchronize()
    ts = [s.elapsed_time(e) * 1e3 for s, e in ev]
    return round(sum(ts) / len(ts), 2), round(min(ts), 2), round(max(ts), 2)
z = torch.zeros(1, device="cuda")
x = torch.randn(2048, 14336, device="cuda").bfloat16()
a = alloc_result(2048, 14336, 0, 32, "cuda")
xs = torch.randn(16, 4096, device="cuda").bfloat16()
b = alloc_result(16, 4096, 0, 32, "cuda")
print(json.dumps({
    "nothing": timeit(lambda: None),
    "add1": timeit(lambda: z.add_(1)),
    "add1_noflush": timeit(lambda: z.add_(1), fl=False),
    "k1_c1": timeit(lambda: act_quant_into(x, 0, 32, a.codes, a.sf, a.tensor_scale_dev, a.scratch)),
    "k1_tiny": timeit(lambda: act_quant_into(xs, 0, 32, b.codes, b.sf, b.tensor_scale_dev, b.scratch)),
    "k1_tiny_noflush": timeit(lambda: act_quant_into(xs, 0, 32, b.codes, b.sf, b.tensor_scale_dev, b.scratch), fl=False),
    "pdl": os.environ.get("MRFP4_PDL", "1")}))
