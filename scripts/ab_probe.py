"""A/B in one process: a debug toggle (argv[1] = exported setter name) off/on, interleaved, on GEMM shapes.
argv[2] == "step" times act-quant + GEMM."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
L = _lib.lib()
setter = getattr(L, sys.argv[1]); setter.argtypes = [ctypes.c_int]
STEP = len(sys.argv) > 2 and sys.argv[2] == "step"  # time K1+K2 (PDL overlap) instead of K2 alone
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")

def timeit(fn, iters=100):
    for _ in range(3): fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for s, e in ev:
        flush.zero_(); flush.sum(dtype=torch.int32); s.record(); fn(); e.record()
    torch.cuda.synchronize()
    ts = [s.elapsed_time(e) for s, e in ev]
    return sum(ts) / len(ts) * 1e3  # mean: event times are quantized (~2 us steps)

for M, K, N, fmt in [(2048, 14336, 4096, 0), (2048, 28672, 8192, 0), (2048, 8192, 28672, 1), (512, 8192, 28672, 0), (8192, 8192, 8192, 0)]:
    spec = P.FormatSpec.mxfp4() if fmt == 0 else P.FormatSpec.nvfp4()
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K**0.5).bfloat16(), spec, None)
    a = alloc_result(M, K, w.fmt, 0, "cuda")
    act_quant_into(x, w.fmt, 0, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    res = {0: [], 1: []}
    for rep in range(3):
        for v in (0, 1):
            setter(v)
            if STEP:
                res[v].append(timeit(lambda: (act_quant_into(x, w.fmt, 0, a.codes, a.sf, a.tensor_scale_dev, a.scratch), P.gemm(a, w, out))))
            else:
                res[v].append(timeit(lambda: P.gemm(a, w, out)))
    setter(1)
    print(json.dumps(dict(M=M, K=K, N=N, fmt=fmt, off=[round(t, 1) for t in res[0]], on=[round(t, 1) for t in res[1]])))
