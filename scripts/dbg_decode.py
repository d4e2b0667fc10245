import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle as O, paper_2509_23202_b200 as P
from test_gpu_decode import two_kernel
for fmt, k, (M, K, N) in (("mxfp4", 32, (16, 4096, 4096)), ("mxfp4", 32, (16, 1024, 256)), ("mxfp4", 0, (16, 1024, 256)), ("nvfp4", 16, (16, 1024, 256)), ("mxfp4", 32, (16, 256, 128))):
    rng = np.random.default_rng(M * 7 + K + N + k)
    X = O.bf16_round(rng.standard_normal((M, K)) * np.exp(rng.uniform(-1, 1, size=(M, 1))))
    W = O.bf16_round(rng.standard_normal((N, K)) / np.sqrt(K))
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    w = P.quantize_weight(torch.from_numpy(W).cuda().bfloat16(), spec, P.TransformSpec.hadamard(k) if k else None)
    x = torch.from_numpy(X).cuda().bfloat16()
    y = P.quantized_linear(x, w, out_dtype=torch.float32).cpu().numpy()
    y2 = two_kernel(x, w, torch.float32).cpu().numpy()
    d = np.abs(y - y2) / (np.abs(y2) + 1e-6)
    bad = np.argwhere(d > 1e-4)
    print(fmt, k, M, K, N, "max rel", d.max(), "n bad", len(bad), "rows", sorted(set(bad[:, 0].tolist()))[:8], "cols", sorted(set(bad[:, 1].tolist()))[:8], "ratio sample", (y[tuple(bad[0])] / y2[tuple(bad[0])]) if len(bad) else None)
