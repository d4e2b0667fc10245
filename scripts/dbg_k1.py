import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2509_23202_b200 as P
for (M,K,fmt,k) in [(8,64,'mxfp4',32),(64,1024,'mxfp4',32),(64,1024,'nvfp4',16),(3,48,'nvfp4',16)]:
    x=torch.randn(M,K,device='cuda').bfloat16()
    spec=P.FormatSpec.mxfp4() if fmt=='mxfp4' else P.FormatSpec.nvfp4()
    r=P.quantize_rtn(x,spec,transform=P.TransformSpec.hadamard(k),check=False)
    torch.cuda.synchronize(); print('ok',M,K,fmt,k, flush=True)
