"""K2 with and without the stream-K tail (flushed L2, event timing) at the bench / sweep shapes."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
L = _lib.lib(); fs = L.mrfp4_debug_gemm_stream_k; fs.argtypes = [ctypes.c_int]
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda"); fr = torch.ones(64 * 2**20, dtype=torch.int32, device="cuda")
def timeit(fn, n=30):
    for _ in range(3): fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for s, e in ev:
        flush.zero_(); fr.sum(dtype=torch.int32); s.record(); fn(); e.record()
    torch.cuda.synchronize()
    return round(sum(s.elapsed_time(e) for s, e in ev) / n * 1e3, 1)
shapes = [(2048, 14336, 4096, "mxfp4")]
shapes += [(M, K, N, f) for (K, N, f) in [(8192, 28672, "nvfp4"), (28672, 8192, "mxfp4")] for M in (512, 1024, 2048, 4096)]
shapes += [(2048, 5120, 51200, "nvfp4")]
for M, K, N, fmt in shapes:
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** .5).bfloat16(), spec, P.TransformSpec.hadamard(16))
    a = alloc_result(M, K, w.fmt, 16, "cuda"); act_quant_into(x, w.fmt, 16, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    r = {}
    for on in (0, 1):
        fs(on); r["sk" if on else "dp"] = timeit(lambda: P.gemm(a, w, y))
        if on: y1 = y.clone()
        else: y0 = y.clone()
    fs(1)
    err = float((y1.float() - y0.float()).norm() / y0.float().norm())
    print(json.dumps(dict(M=M, K=K, N=N, fmt=fmt, **r, rel=round(err, 6))))
