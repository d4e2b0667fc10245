"""Host wall-clock per layer call at decode sizes: eager quantized_linear vs GraphedLinear."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
for (M, K, N, fmt, k) in [(16, 4096, 4096, "nvfp4", 16), (1, 8192, 28672, "nvfp4", 16), (16, 28672, 8192, "mxfp4", 32)]:
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** .5).bfloat16(), spec, P.TransformSpec.hadamard(k))
    x = torch.randn(M, K, device="cuda").bfloat16()
    g = P.GraphedLinear(w, M)
    g.x.copy_(x)
    def rate(fn, n=2000):
        for _ in range(50): fn()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(n): fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / n * 1e6
    print(json.dumps(dict(M=M, K=K, N=N, fmt=fmt, eager_us=round(rate(lambda: P.quantized_linear(x, w)), 1),
                          graph_us=round(rate(lambda: g()), 1))))
