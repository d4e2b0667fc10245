import ctypes, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from paper_2509_23202_b200 import _lib
from test_gpu_gemm import random_container, run_gemm, ref64, rel_fro
L = _lib.lib(); fd = L.mrfp4_debug_gemm_mode; fd.argtypes = [ctypes.c_int]
for (M, N, K) in [(256, 256, 16384), (512, 512, 8192), (8192, 8192, 1024), (2048, 4096, 4096), (2048, 4096, 14336)]:
    for fmt in ("mxfp4", "nvfp4"):
        rng = np.random.default_rng(M + N + K)
        A, W = random_container(rng, M, K, fmt), random_container(rng, N, K, fmt)
        ref = ref64(A, W)
        out = []
        for mode in (0, 200 + 1, 200 + 0):
            fd(mode); y = run_gemm(A, W).cpu().numpy(); fd(0)
            out.append(round(rel_fro(y, ref), 7))
        print(M, N, K, fmt, "ahead=S / 1 / 0:", out)
