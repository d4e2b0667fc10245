"""K2 experiments: normal vs no-load vs no-MMA timing at a few shapes (device events, L2 flushed)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into

L = _lib.lib()
L.mrfp4_debug_gemm_mode.argtypes = [ctypes.c_int]
L.mrfp4_debug_gemm_kernel.argtypes = [ctypes.c_int]
KERNEL = int(os.environ.get("KERNEL", "0"))
L.mrfp4_debug_gemm_kernel(KERNEL)
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")

def timeit(fn, iters=20, warm=3):
    for _ in range(warm): fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort(); return ts[len(ts)//2] * 1e-3

import subprocess
subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw", "--format=csv"])
for M, K, N, fmt in [(2048, 14336, 4096, "mxfp4"), (4096, 8192, 8192, "nvfp4"), (8192, 8192, 8192, "mxfp4")]:
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K**0.5).bfloat16(), spec, None)
    a = alloc_result(M, K, w.fmt, 0, "cuda")
    act_quant_into(x, w.fmt, 0, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    res = {}
    for mode in (0, 1, 64):
        L.mrfp4_debug_gemm_mode(mode)
        t = timeit(lambda: P.gemm(a, w, out))
        res[mode] = (t * 1e6, 2 * M * N * K / t / 1e12)
    L.mrfp4_debug_gemm_mode(0)
    print(json.dumps(dict(M=M, K=K, N=N, fmt=fmt, normal=res[0], no_ld=res[1], no_mma=res[64])), flush=True)
