"""Wall clock of the GPU MR-GPTQ solver on a full Qwen3-32B linear (default: down_proj,
N=5120 x K=25600, NVFP4 + H128, MSE scales, act-order), then the layer through the GEMM."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import gptq as G

N, K = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (5120, 25600)))
k = int(sys.argv[3]) if len(sys.argv) > 3 else 128
g = torch.Generator(device="cuda").manual_seed(0)
W = torch.randn(N, K, generator=g, device="cuda", dtype=torch.float64) / K ** 0.5
H = G.Hessian(K)
G.accumulate_hessian(torch.randn(512, K, generator=g, device="cuda", dtype=torch.float64), H)
torch.cuda.synchronize()
t0 = time.time()
res = G.mr_gptq(W, H, P.FormatSpec.nvfp4(), transform=P.TransformSpec.hadamard(k))
torch.cuda.synchronize()
t1 = time.time()
w = P.prepare_weight(res)
y = P.quantized_linear(torch.randn(2048, K, device="cuda").bfloat16(), w)
torch.cuda.synchronize()
print(f"mr_gptq NVFP4+H{k} {N}x{K}: {t1 - t0:.1f} s wall (mse_rel {res.mse_rel:.5f}); GEMM output finite: "
      f"{bool(torch.isfinite(y).all())}")
