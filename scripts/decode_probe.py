"""c0 decode (16x4096->4096 NVFP4+H16): K1 alone, K2 alone and K1+K2, flushed L2, event timing;
plus the same without the flush (weights L2-resident, as across a decode loop's layers is not)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda"); fr = torch.ones(64 * 2**20, dtype=torch.int32, device="cuda")
def timeit(fn, n=50, fl=True):
    for _ in range(5): fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for s, e in ev:
        if fl: flush.zero_(); fr.sum(dtype=torch.int32)
        s.record(); fn(); e.record()
    torch.cuda.synchronize()
    t = sorted(s.elapsed_time(e) * 1e3 for s, e in ev)
    return round(t[len(t) // 2], 1)
for M, K, N, fmt, hk in [(16, 4096, 4096, "nvfp4", 16), (16, 4096, 4096, "mxfp4", 32), (1, 4096, 4096, "nvfp4", 16), (64, 4096, 4096, "nvfp4", 16)]:
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** .5).bfloat16(), spec, P.TransformSpec.hadamard(hk))
    a = alloc_result(M, K, w.fmt, hk, "cuda")
    k1 = lambda: act_quant_into(x, w.fmt, hk, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    k1()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    k2 = lambda: P.gemm(a, w, y)
    wb = w.N * w.K
    bf = torch.randn(N, K, device="cuda").bfloat16()
    cub = lambda: torch.mm(x, bf.t())
    r = dict(k1=timeit(k1), k2=timeit(k2), both=timeit(lambda: (k1(), k2())), cublas=timeit(cub),
             k1_warm=timeit(k1, fl=False), k2_warm=timeit(k2, fl=False), both_warm=timeit(lambda: (k1(), k2()), fl=False),
             cublas_warm=timeit(cub, fl=False))
    print(M, K, N, fmt, r, flush=True)

# Warm GPU time per call: 20 back-to-back calls captured in one CUDA graph (no host gaps).
def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps): fn()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [g.replay() for _ in range(10)]; e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / (10 * reps), 2)
for M, K, N, fmt, hk in [(16, 4096, 4096, "nvfp4", 16), (16, 4096, 4096, "mxfp4", 32)]:
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** .5).bfloat16(), spec, P.TransformSpec.hadamard(hk))
    a = alloc_result(M, K, w.fmt, hk, "cuda")
    k1 = lambda: act_quant_into(x, w.fmt, hk, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    k2 = lambda: P.gemm(a, w, y)
    bf = torch.randn(N, K, device="cuda").bfloat16()
    print("graph-warm", M, fmt, dict(k1=graph_time(k1), k2=graph_time(k2), both=graph_time(lambda: (k1(), k2())),
                                      cublas=graph_time(lambda: torch.mm(x, bf.t()))), flush=True)
