import ctypes, os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import torch
from test_gpu_fullsize import SHAPES, operands, dequant, alloc_result, act_quant_into, P
from paper_2509_23202_b200 import _lib
L = _lib.lib(); fd = L.mrfp4_debug_gemm_mode; fd.argtypes = [ctypes.c_int]
M, K, N, fmt, k = SHAPES["c4"]
x, w = operands("c4")
a = alloc_result(M, K, w.fmt, k, "cuda")
act_quant_into(x, w.fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
da = dequant(a.codes, a.sf, a.tensor_scale_dev, M, K, w.fmt)
cb = K // 16 // 4
n0, nn = 8192, 16384
dw = dequant(w.codes[n0:n0 + nn], w.sf[(n0 // 128) * cb * 512:], w.tensor_scale_dev, nn, K, w.fmt)
ref = (da.double() @ dw.double().T)
for mode in (0, 32, 16, 32, 16):
    fd(mode)
    y = torch.empty((M, N), dtype=torch.float32, device="cuda")
    P.gemm(a, w, y); torch.cuda.synchronize()
    e = (y[:, n0:n0 + nn].double() - ref).abs() > 1e-3
    print("mode", mode, "bad rows", int(e.any(dim=1).sum()))
fd(0)
