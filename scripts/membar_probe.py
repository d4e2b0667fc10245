"""MXFP4 K2: is the forwarder's membar costly by its latency on the path or by its presence?
debug 0: release arrival (correct); 77: relaxed arrival then membar (racy, membar off-path);
78: relaxed only (racy)."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
L = _lib.lib(); fd = L.mrfp4_debug_gemm_mode; fd.argtypes = [ctypes.c_int]
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda"); fr = torch.ones(64 * 2**20, dtype=torch.int32, device="cuda")
def timeit(fn, n=30):
    for _ in range(3): fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for s, e in ev:
        flush.zero_(); fr.sum(dtype=torch.int32); s.record(); fn(); e.record()
    torch.cuda.synchronize()
    return round(sum(s.elapsed_time(e) for s, e in ev) / n * 1e3, 1)
for M, K, N in [(2048, 14336, 4096), (2048, 28672, 8192)]:
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** .5).bfloat16(), P.FormatSpec.mxfp4(), P.TransformSpec.hadamard(32))
    a = alloc_result(M, K, w.fmt, 32, "cuda"); act_quant_into(x, w.fmt, 32, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    r = {}
    for mode in (0, 77, 78):
        fd(mode); r[mode] = timeit(lambda: P.gemm(a, w, y))
    fd(0)
    print(json.dumps(dict(M=M, K=K, N=N, **{str(k): v for k, v in r.items()})))
