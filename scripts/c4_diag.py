import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import torch
from test_gpu_fullsize import SHAPES, operands, dequant, alloc_result, act_quant_into, P
name = "c4"
M, K, N, fmt, k = SHAPES[name]
x, w = operands(name)
a = alloc_result(M, K, w.fmt, k, "cuda")
act_quant_into(x, w.fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
y = torch.empty((M, N), dtype=torch.float32, device="cuda")
P.gemm(a, w, y)
da = dequant(a.codes, a.sf, a.tensor_scale_dev, M, K, w.fmt)
cb = K // 16 // 4
rows = torch.arange(0, M, 37, device="cuda")
for n0 in range(0, N, 4096):
    nn = min(4096, N - n0)
    dw = dequant(w.codes[n0:n0 + nn], w.sf[(n0 // 128) * cb * 512:], w.tensor_scale_dev, nn, K, w.fmt)
    ref64 = da[rows].double() @ dw.double().T
    yy = y[rows, n0:n0 + nn].double()
    e = (yy - ref64)
    rel = float(e.norm() / ref64.norm())
    bad_rows = (e.abs() > 1e-3).any(dim=1).nonzero().flatten()
    print(n0, round(rel, 9), "bad rows:", rows[bad_rows][:8].tolist(), "bad m-blocks:", sorted(set((rows[bad_rows] // 256).tolist()))[:10])
