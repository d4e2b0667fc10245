"""Small invocations of every kernel family for compute-sanitizer (scripts/sanitize.sh):
K1 (MXFP4 single pass, NVFP4 two-phase grid barrier, NVFP4 static s_T, butterfly fp32 path),
K2 (1-CTA split-K with in-kernel reduction, 2-CTA cta_group::2), the one-kernel decode linear
(M <= 32: cluster DSMEM st.async exchanges), the requant epilogue, the float64 path, the GPTQ
block solver.  Prints one line per case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import gptq as G

torch.manual_seed(0)
MX, NV = P.FormatSpec.mxfp4(), P.FormatSpec.nvfp4()
for spec, k in ((MX, 32), (NV, 16)):
    tr = P.TransformSpec.hadamard(k)
    W = (torch.randn(512, 1024, device="cuda") / 32).bfloat16()
    w = P.quantize_weight(W, spec, tr)
    for M in (1, 16, 32, 100, 300):   # 1/16/32: k_linear_decode; 100: 1-CTA K2; 300: 2-CTA K2
        x = torch.randn(M, 1024, device="cuda").bfloat16()
        y = P.quantized_linear(x, w, check=True)
        torch.cuda.synchronize()
        print(f"linear {spec.group_size} M={M}: ok {bool(torch.isfinite(y).all())}")
    r = P.quantize_rtn(torch.randn(64, 1024, device="cuda").float(), spec, transform=tr)   # butterfly path
    print(f"fp32 K1 {spec.group_size}: ok")
for spec, k in ((MX, 32), (NV, 16)):   # M = 24: two activation segments per thread
    w = P.quantize_weight((torch.randn(1024, 4096, device="cuda") / 64).bfloat16(), spec, P.TransformSpec.hadamard(k))
    y = P.quantized_linear(torch.randn(24, 4096, device="cuda").bfloat16(), w, check=True)
    torch.cuda.synchronize()
    print(f"decode 2-seg {spec.group_size}: ok {bool(torch.isfinite(y).all())}")
for spec, k in ((MX, 128), (NV, 64)):   # cross-lane Hadamard stages in the decode kernel
    w = P.quantize_weight((torch.randn(512, 1024, device="cuda") / 32).bfloat16(), spec, P.TransformSpec.hadamard(k))
    y = P.quantized_linear(torch.randn(16, 1024, device="cuda").bfloat16(), w, check=True)
    torch.cuda.synchronize()
    print(f"decode H{k} {spec.group_size}: ok {bool(torch.isfinite(y).all())}")
for spec, k in ((MX, 32), (NV, 16), (NV, 128)):   # wide weight: the persistent decode variant (k_linear_decode_p)
    w = P.quantize_weight((torch.randn(20480, 1024, device="cuda") / 32).bfloat16(), spec, P.TransformSpec.hadamard(k))
    for M in (1, 4):
        y = P.quantized_linear(torch.randn(M, 1024, device="cuda").bfloat16(), w, check=True)
        torch.cuda.synchronize()
        print(f"wide linear {spec.group_size} M={M}: ok {bool(torch.isfinite(y).all())}")
st = P.quantize_rtn(torch.randn(64, 1024, device="cuda").bfloat16(), NV, static_tensor_scale=0.002)
x = torch.randn(300, 1024, device="cuda").bfloat16()
w = P.quantize_weight((torch.randn(512, 1024, device="cuda") / 32).bfloat16(), MX, P.TransformSpec.hadamard(32))
q = P.quantized_linear_requant(x, w, P.TransformSpec.hadamard(32), check=True)
q2 = P.quantized_linear_requant(x, w, P.TransformSpec.hadamard(16), next_spec=NV, next_tensor_scale=0.01)
r64 = P.quantize_rtn(torch.randn(8, 256, device="cuda", dtype=torch.float64), NV, transform=P.TransformSpec.hadamard(16))
H = G.accumulate_hessian(torch.randn(64, 256, device="cuda", dtype=torch.float64), G.Hessian(256))
g = G.mr_gptq(torch.randn(32, 256, device="cuda", dtype=torch.float64), H, NV)
torch.cuda.synchronize()
print("requant / static / f64 / gptq: ok")
