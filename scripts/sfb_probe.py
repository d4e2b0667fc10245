"""Which CTA's TMEM does the cta_group::2 block-scaled MMA read SFB from?  (debug 64: peer SFB
zeroed; 65: peer keeps only block 1; 66: leader keeps only block 0)."""
import ctypes, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2509_23202_b200 as P
from paper_2509_23202_b200 import _lib
from test_gpu_gemm import random_container, run_gemm, ref64, rel_fro
L = _lib.lib(); fd = L.mrfp4_debug_gemm_mode; fd.argtypes = [ctypes.c_int]
for fmt in ("mxfp4", "nvfp4"):
    rng = np.random.default_rng(3)
    A, W = random_container(rng, 512, 1024, fmt), random_container(rng, 512, 1024, fmt)
    ref = ref64(A, W)
    for mode in (0, 64, 65, 66):
        fd(mode)
        y = run_gemm(A, W).cpu().numpy()
        fd(0)
        bad = np.abs(y - ref) > 1e-3 * np.abs(ref).max()
        print(fmt, mode, "rel", rel_fro(y, ref), "bad cols (mod 256) sample", sorted(set((np.nonzero(bad)[1] % 256 // 64).tolist())), "bad rows mod 256 //128", sorted(set((np.nonzero(bad)[0] % 256 // 128).tolist())))
