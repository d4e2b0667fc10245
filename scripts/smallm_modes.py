"""1-CTA (split-K) K2 at decode-sized M on the 70B up/down weights, by debug mode (MRFP4_TRACE
build): 0 normal, 1 no operand loads, 2 no MMAs -- is the weight stream or the MMA chain the limit?"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import act_quant_into, alloc_result
from paper_2509_23202_b200.linear import gemm_workspace_bytes
L = _lib.lib(); L.mrfp4_debug_gemm_mode.argtypes = [ctypes.c_int]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, n=20):
    for _ in range(3): fn()
    ev = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    return sum(x.elapsed_time(y) for x, y in ev) / n * 1e3
for (K, N) in ((8192, 28672), (28672, 8192)):
    spec = P.FormatSpec.mxfp4()
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16(), spec, P.TransformSpec.hadamard(32))
    wb = N * K * (0.5 + 1 / 32)
    for M in (16, 128):
        x = torch.randn(M, K, device="cuda").bfloat16()
        a = alloc_result(M, K, w.fmt, 32, "cuda")
        act_quant_into(x, w.fmt, 32, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
        y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        ws = torch.zeros(max(gemm_workspace_bytes(M, w), 1), dtype=torch.uint8, device="cuda")
        out = []
        for mode in (0, 1, 2):
            L.mrfp4_debug_gemm_mode(mode)
            us = t(lambda: P.gemm(a, w, y, ws))
            out.append(f"mode{mode} {us:.1f} us ({wb / us / 1e3:.0f} GB/s)")
        L.mrfp4_debug_gemm_mode(0)
        print(f"K={K} N={N} M={M}:", "  ".join(out))
