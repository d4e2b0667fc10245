"""K2 at M in {64, 128, 192, 256} for the 70B shapes: the 1-CTA split-K kernel vs the 2-CTA kernel
forced (mrfp4_debug_gemm_kernel), flushed L2, CUDA events."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import act_quant_into, alloc_result
from paper_2509_23202_b200.linear import gemm_workspace_bytes
L = _lib.lib(); fk = L.mrfp4_debug_gemm_kernel; fk.argtypes = [ctypes.c_int]; fk.restype = ctypes.c_int
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, n=30):
    for _ in range(3): fn()
    ev = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    return sum(x.elapsed_time(y) for x, y in ev) / n * 1e3
for (K, N) in ((8192, 28672), (28672, 8192)):
    for fmt, had, spec in (("nvfp4", 16, P.FormatSpec.nvfp4()), ("mxfp4", 32, P.FormatSpec.mxfp4())):
        w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16(), spec, P.TransformSpec.hadamard(had))
        for M in (64, 128, 192, 256):
            x = torch.randn(M, K, device="cuda").bfloat16()
            a = alloc_result(M, K, w.fmt, had, "cuda")
            act_quant_into(x, w.fmt, had, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
            y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            ws = torch.zeros(max(gemm_workspace_bytes(M, w), 1), dtype=torch.uint8, device="cuda")
            res = {}
            for kern in (1, 2):
                fk(kern)
                try:
                    res[kern] = t(lambda: P.gemm(a, w, y, ws))
                except Exception as e:
                    res[kern] = float("nan")
            fk(0)
            print(f"K={K} N={N} {fmt} M={M}: 1-CTA {res[1]:.1f} us  2-CTA {res[2]:.1f} us")
