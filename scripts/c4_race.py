"""c4 GEMM: which rows go wrong, and does it depend on PDL / weight pre-issue / output dtype?"""
import ctypes, os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import torch
from test_gpu_fullsize import SHAPES, operands, dequant, alloc_result, act_quant_into, P
from paper_2509_23202_b200 import _lib
L = _lib.lib(); L.mrfp4_debug_gemm_preissue.argtypes = [ctypes.c_int]
M, K, N, fmt, k = SHAPES["c4"]
x, w = operands("c4")
a = alloc_result(M, K, w.fmt, k, "cuda")
act_quant_into(x, w.fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
torch.cuda.synchronize()
da = dequant(a.codes, a.sf, a.tensor_scale_dev, M, K, w.fmt)
cb = K // 16 // 4
n0, nn = 8192, 16384
dw = dequant(w.codes[n0:n0 + nn], w.sf[(n0 // 128) * cb * 512:], w.tensor_scale_dev, nn, K, w.fmt)
ref = (da.double() @ dw.double().T)   # rows all, cols [n0, n0+nn)
def bad(y):
    e = (y[:, n0:n0 + nn].double() - ref).abs() > 1e-3
    r = e.any(dim=1).nonzero().flatten()
    return len(r), r[:6].tolist()
for tag, pre, dt in [("default bf16", 1, torch.bfloat16), ("default f32", 1, torch.float32), ("default f32 again", 1, torch.float32),
                     ("no preissue f32", 0, torch.float32), ("no preissue f32 again", 0, torch.float32)]:
    L.mrfp4_debug_gemm_preissue(pre)
    y = torch.empty((M, N), dtype=dt, device="cuda")
    P.gemm(a, w, y)
    torch.cuda.synchronize()
    print(tag, bad(y.float()))
L.mrfp4_debug_gemm_preissue(1)
