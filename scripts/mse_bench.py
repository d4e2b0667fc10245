"""GPU MSE scale search throughput (offline weight quantization).
Wall clock per call (the search syncs: its group-error totals are summed with numpy)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_23202_b200 as P
pol = P.ScalePolicy(mode=P.ScaleMode.MSE)
for (N, K, fmt, k) in [(512, 4096, "nvfp4", 16), (4096, 4096, "nvfp4", 16), (4096, 4096, "mxfp4", 32), (8192, 28672, "nvfp4", 16)]:
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    P.quantize(W[:256], spec, policy=pol, transform=P.TransformSpec.hadamard(k))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = P.quantize(W, spec, policy=pol, transform=P.TransformSpec.hadamard(k))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps(dict(N=N, K=K, fmt=fmt, k=k, seconds=round(dt, 3), melem_per_s=round(N * K / dt / 1e6, 1),
                          mse_rel=r.mse_rel)))
