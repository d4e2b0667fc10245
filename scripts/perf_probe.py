"""Quick device timings of K1 / K2 / cuBLAS bf16 at a few shapes (CUDA events, L2-flushed)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200.quantize import alloc_result, act_quant_into

torch.manual_seed(0)
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")

def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2] * 1e-3

shapes = [(2048, 14336, 4096, "mxfp4", 32), (16, 4096, 4096, "nvfp4", 16), (8192, 8192, 28672, "nvfp4", 16),
          (512, 8192, 28672, "mxfp4", 32), (2048, 28672, 8192, "nvfp4", 16), (8192, 28672, 8192, "mxfp4", 32)]
for M, K, N, fmt, k in shapes:
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    tr = P.TransformSpec.hadamard(k)
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = P.quantize_weight((torch.randn(N, K, device="cuda") / K**0.5).bfloat16(), spec, tr)
    a = alloc_result(M, K, w.fmt, k, "cuda")
    out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    t1 = timeit(lambda: act_quant_into(x, w.fmt, k, a.codes, a.sf, a.tensor_scale_dev, a.scratch))
    t2 = timeit(lambda: P.gemm(a, w, out))
    wb = torch.randn(N, K, device="cuda").bfloat16()
    t3 = timeit(lambda: torch.matmul(x, wb.t()))
    G = 32 if fmt == "mxfp4" else 16
    k1_bytes = M * K * (2 + 0.5 + 1 / G)
    fl = 2 * M * N * K
    print(json.dumps(dict(M=M, K=K, N=N, fmt=fmt, k=k, k1_us=t1 * 1e6, k1_gbs=k1_bytes / t1 / 1e9,
                          k2_us=t2 * 1e6, k2_tflops=fl / t2 / 1e12, bf16_us=t3 * 1e6, bf16_tflops=fl / t3 / 1e12,
                          speedup=t3 / (t1 + t2))))
