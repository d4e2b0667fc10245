"""C3 weight fixtures from the REAL reference MR-GPTQ solver, as BASELINE.json configs[3] writes it:
Qwen3-32B decoder-layer linears, MR-GPTQ-quantized, Hadamard-128, NVFP4.

Usage (dev container only; /root/reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c3.py

For each linear (QKV 5120->10240, O 8192->5120, gate-up 5120->51200, down 25600->5120) a
128-row slice of a random N(0, 1/K) weight is quantized by the unmodified
``mr_gptq(W, H, FormatSpec.nvfp4(), transform=TransformSpec.hadamard(128))`` (gptq.py:274-300:
conjugated Hessian, MSE-searched E4M3 scales, static act-order, lazy-block Cholesky solve) at
the layer's FULL K, against a Hessian of 512 Gaussian calibration rows.
The CPU solver is infeasible at full N (42.6 s per 256x4096 slice), so the GPU tests tile the
slice to the layer's full N for the GEMM and check parity on the slice itself.

Writes ``tests/golden/c3_mrgptq.npz``: per layer the packed codes, row-major E4M3 scale codes,
tensor scale and the reference's mse_rel of the slice.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

from microfp import FormatSpec, TransformSpec  # noqa: E402
from microfp.gptq import Hessian, accumulate_hessian, mr_gptq  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
LAYERS = {  # name: (K, N) of Qwen3-32B (hidden 5120, 64 q heads x 128 + 2 x 8 kv heads x 128, ffn 25600)
    "qkv": (5120, 10240),
    "o": (8192, 5120),
    "gateup": (5120, 51200),
    "down": (25600, 5120),
}
ROWS, CALIB = 128, 512


def main(names):
    out = {}
    path = os.path.join(HERE, "c3_mrgptq.npz")
    if os.path.exists(path):
        out = dict(np.load(path))
    for name in names:
        K, N = LAYERS[name]
        rng = np.random.default_rng(3202 + list(LAYERS).index(name))
        W = rng.standard_normal((ROWS, K)) / np.sqrt(K)
        H = accumulate_hessian(rng.standard_normal((CALIB, K)), Hessian(K))
        t0 = time.time()
        res = mr_gptq(W, H, FormatSpec.nvfp4(), transform=TransformSpec.hadamard(128))
        t = res.tensor
        out[f"{name}_codes"] = np.asarray(t.codes, dtype=np.uint8)
        out[f"{name}_scales"] = np.asarray(t.scale_codes, dtype=np.uint8)
        out[f"{name}_ts"] = np.float64(t.tensor_scale)
        out[f"{name}_shape"] = np.array([ROWS, K, N], dtype=np.int64)
        out[f"{name}_mse_rel"] = np.float64(res.mse_rel)
        print(f"{name}: K={K} {time.time() - t0:.1f} s ts={t.tensor_scale:.6g} mse_rel={res.mse_rel:.4g}", flush=True)
        np.savez_compressed(path, **out)


if __name__ == "__main__":
    main(sys.argv[1:] or list(LAYERS))
