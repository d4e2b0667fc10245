"""Launch cuBLASLt's NVFP4 GEMM (torch._scaled_mm) on c2-up operands a few times (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2509_23202_b200 as P
from paper_2509_23202_b200.quantize import act_quant_into, alloc_result
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2-up-nv"
name, M, K, N, fmt, had = bench.CONFIGS[cfg]
x = torch.randn(M, K, device="cuda").bfloat16()
w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16(), P.FormatSpec.nvfp4(), P.TransformSpec.hadamard(had))
a = alloc_result(M, K, w.fmt, had, "cuda")
act_quant_into(x, w.fmt, had, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
a4, b4 = a.codes.view(torch.float4_e2m1fn_x2), w.codes.view(torch.float4_e2m1fn_x2)
for _ in range(5):
    y = torch._scaled_mm(a4, b4.t(), a.sf.view(torch.float8_e4m3fn), w.sf.view(torch.float8_e4m3fn), out_dtype=torch.bfloat16)
torch.cuda.synchronize()
print("ok", y.shape)
