"""Fused next-layer quantization (K2 epilogue) vs K2 + a separate K1 on its bf16 output."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda"); fr = torch.ones(64 * 2**20, dtype=torch.int32, device="cuda")
def timeit(fn, n=40):
    for _ in range(3): fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for s, e in ev:
        flush.zero_(); fr.sum(dtype=torch.int32); s.record(); fn(); e.record()
    torch.cuda.synchronize()
    return round(sum(s.elapsed_time(e) for s, e in ev) / n * 1e3, 1)
L = _lib.lib()
for M, K, N, fmt in [(2048, 14336, 4096, "mxfp4"), (2048, 4096, 14336, "mxfp4"), (8192, 8192, 28672, "mxfp4")]:
    spec = P.FormatSpec.mxfp4()
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** .5).bfloat16(), spec, P.TransformSpec.hadamard(32))
    a = alloc_result(M, K, w.fmt, 32, "cuda"); act_quant_into(x, w.fmt, 32, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    nxt = alloc_result(M, N, 0, 32, "cuda")
    def unfused():
        P.gemm(a, w, y)
        act_quant_into(y, 0, 32, nxt.codes, nxt.sf, nxt.tensor_scale_dev, nxt.scratch)
    def fused(store_y):
        st = _lib.stream_ptr(torch, y.device)
        _lib.check(L.mrfp4_gemm_quant_next(_lib.ptr(a.codes), _lib.ptr(a.sf), _lib.ptr(a.tensor_scale_dev),
            _lib.ptr(w.codes), _lib.ptr(w.sf), _lib.ptr(w.tensor_scale_dev), _lib.ptr(y) if store_y else None, N, M, N, K,
            w.fmt, 32, _lib.ptr(nxt.codes), _lib.ptr(nxt.sf), _lib.ptr(nxt.tensor_scale_dev), _lib.ptr(nxt.scratch), st))
    r = dict(M=M, K=K, N=N, k2=timeit(lambda: P.gemm(a, w, y)), k2_plus_k1=timeit(unfused),
             fused=timeit(lambda: fused(False)), fused_keep_y=timeit(lambda: fused(True)))
    print(json.dumps(r))
