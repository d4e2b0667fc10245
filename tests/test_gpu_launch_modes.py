"""Launch-mode switches give bit-identical results: MRFP4_COOP=1 (cooperative launches for the
kernels that synchronize their own CTAs: NVFP4's two-phase K1, the split-K GEMM), MRFP4_PDL=0
(no programmatic dependent launch) and MRFP4_DECODE=0 (decode shapes through K1 + K2 instead of
the one-kernel decode linear, within fp32 summation order).  Each mode runs in its own process
(the switches are read once per process)."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2509_23202_b200 as P
torch.manual_seed(0)
out = []
for spec, k in ((P.FormatSpec.nvfp4(), 16), (P.FormatSpec.mxfp4(), 32)):
    w = P.quantize_weight((torch.randn(1024, 2048, device="cuda") / 45).bfloat16(), spec, P.TransformSpec.hadamard(k))
    for M in (16, 64, 300):   # decode kernel / K1 + split-K K2 / K1 + 2-CTA K2
        x = torch.randn(M, 2048, device="cuda").bfloat16()
        out.append(P.quantized_linear(x, w, out_dtype=torch.float32, check=True).cpu().numpy())
np.savez(sys.argv[2], *out)
"""


def run_mode(tmp_path, name, env_extra):
    path = tmp_path / f"{name}.npz"
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(path)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    z = np.load(path)
    return [z[f"arr_{i}"] for i in range(len(z.files))]


def test_launch_modes_agree(tmp_path):
    base = run_mode(tmp_path, "default", {})
    for name, env in (("coop", {"MRFP4_COOP": "1"}), ("nopdl", {"MRFP4_PDL": "0"})):
        for a, b in zip(base, run_mode(tmp_path, name, env)):
            assert np.array_equal(a, b), name
    two = run_mode(tmp_path, "nodecode", {"MRFP4_DECODE": "0"})
    for i, (a, b) in enumerate(zip(base, two)):
        if i % 3 == 0:   # the M = 16 cases: same codes, different fp32 summation order
            assert np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(b)
        else:
            assert np.array_equal(a, b)
