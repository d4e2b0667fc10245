"""Is the flushed event timing host-launch bound?  Same kernels, with and without a GPU-side
spin (torch.cuda._sleep) between the L2 flush and the start event, so the host can queue
the timed launches before the GPU reaches them."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda"); fr = torch.ones(64 * 2**20, dtype=torch.int32, device="cuda")
def timeit(fn, spin, n=40):
    for _ in range(3): fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for s, e in ev:
        flush.zero_(); fr.sum(dtype=torch.int32)
        if spin: torch.cuda._sleep(spin)
        s.record(); fn(); e.record()
    torch.cuda.synchronize()
    return round(sum(s.elapsed_time(e) for s, e in ev) / n * 1e3, 2)
for M, K, N, fmt, k in [(1, 8192, 28672, "nvfp4", 16), (16, 4096, 4096, "nvfp4", 16), (1, 28672, 8192, "mxfp4", 32)]:
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** .5).bfloat16(), spec, P.TransformSpec.hadamard(k))
    a = alloc_result(M, K, w.fmt, k, "cuda")
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    k1 = lambda: act_quant_into(x, w.fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    k2 = lambda: P.gemm(a, w, y)
    def step(): k1(); k2()
    cub = lambda: torch.matmul(x, torch.empty(0, device="cuda") if False else wb.t(), out=yb)
    wb = (torch.randn(N, K, device="cuda") / K ** .5).bfloat16(); yb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    r = {}
    for spin in (0, 200000):
        tag = "spin" if spin else "plain"
        r[f"k1_{tag}"] = timeit(k1, spin); r[f"k2_{tag}"] = timeit(k2, spin); r[f"step_{tag}"] = timeit(step, spin)
        r[f"cublas_{tag}"] = timeit(lambda: torch.matmul(x, wb.t(), out=yb), spin)
    print(json.dumps(dict(M=M, K=K, N=N, **r)))
