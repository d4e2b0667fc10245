"""c0 decode in a CUDA graph, warm (no L2 flush between calls): 20 back-to-back calls of the
one-kernel decode linear (K1 + K2 fused, mrfp4_linear_decode) vs 20 cuBLAS bf16 matmuls of the
same layer, per-call time from graph replays (>= 1.3x warm in a graph).
Also: 20 DIFFERENT layers' weights in sequence (L2 cold per layer, the realistic decode)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2509_23202_b200 as P
from paper_2509_23202_b200.linear import _linear_decode, decode_workspace_bytes


def graph_time(fn, reps=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


res = {}
for fmt, had, M, K, N in (("nvfp4", 16, 16, 4096, 4096), ("mxfp4", 32, 16, 4096, 4096), ("nvfp4", 16, 1, 4096, 4096)):
    spec = P.FormatSpec.nvfp4() if fmt == "nvfp4" else P.FormatSpec.mxfp4()
    L = 20
    wd = [(torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16() for _ in range(L)]
    ws_ = [P.quantize_weight(w, spec, P.TransformSpec.hadamard(had)) for w in wd]
    x = torch.randn(M, K, device="cuda").bfloat16()
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    yb = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    dws = torch.zeros(max(decode_workspace_bytes(M, ws_[0]), 1), dtype=torch.uint8, device="cuda")
    same_ours = graph_time(lambda: [_linear_decode(x, ws_[0], y, dws, None) for _ in range(L)]) / L
    same_bf16 = graph_time(lambda: [torch.matmul(x, wd[0].t(), out=yb) for _ in range(L)]) / L
    diff_ours = graph_time(lambda: [_linear_decode(x, w, y, dws, None) for w in ws_]) / L
    diff_bf16 = graph_time(lambda: [torch.matmul(x, w.t(), out=yb) for w in wd]) / L
    res[f"{fmt} H{had} M={M} {K}->{N}"] = {
        "same_layer_warm_us": {"ours": same_ours, "cublas_bf16": same_bf16, "speedup": same_bf16 / same_ours},
        "20_layers_us": {"ours": diff_ours, "cublas_bf16": diff_bf16, "speedup": diff_bf16 / diff_ours}}
print(json.dumps(res, indent=1))
