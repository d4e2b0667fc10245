"""GPTQ / MR-GPTQ fixtures from the REAL reference solver at the size the verdict names
(256 x 4096 slices), for the GPU solver's parity test (tests/test_gpu_gptq.py).

Usage (dev container only; /root/reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_gptq.py

The weight W [256, 4096] ~ N(0, 1/K) and the calibration batch Xc [512, 4096] ~ N(0, 1) come
from ``np.random.default_rng(SEED)`` in that order, so the test regenerates them.  Stored per
case: packed codes, scale codes, tensor scale, mse_rel, and the reference's proxy loss
(gptq.py:303-311) in the rotated domain: proxy_loss(W H, dequantize(Q), conj(H)), which equals
proxy_loss(W, W_hat, H) (test_gptq.py:263-275).
"""

from __future__ import annotations

import os
import time

import numpy as np

from microfp import FormatSpec, GptqConfig, ScalePolicy, TransformSpec, dequantize  # noqa: E402
from microfp.gptq import Hessian, accumulate_hessian, conjugated_hessian, gptq_quantize, mr_gptq, proxy_loss  # noqa: E402
from microfp.transforms import apply_blockwise  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SEED, ROWS, K, CALIB = 4096, 256, 4096, 512


def inputs():
    rng = np.random.default_rng(SEED)
    W = rng.standard_normal((ROWS, K)) / np.sqrt(K)
    Xc = rng.standard_normal((CALIB, K))
    return W, Xc


def main():
    W, Xc = inputs()
    H = accumulate_hessian(Xc, Hessian(K))
    cases = {
        "mrgptq_nvfp4_h16": lambda: mr_gptq(W, H, FormatSpec.nvfp4()),
        "gptq_mxfp4_h32_absmax": lambda: gptq_quantize(W, H, FormatSpec.mxfp4(), GptqConfig(
            act_order=True, transform=TransformSpec.hadamard(32), scale_policy=ScalePolicy())),
        "gptq_nvfp4_noact_absmax": lambda: gptq_quantize(W, H, FormatSpec.nvfp4(), GptqConfig()),
    }
    out = {}
    for name, fn in cases.items():
        t0 = time.time()
        res = fn()
        t = res.tensor
        tr = t.transform
        Wt = apply_blockwise(W, tr) if tr is not None else W
        Hc = conjugated_hessian(H.matrix, tr) if tr is not None else H.matrix
        loss = proxy_loss(Wt, dequantize(t), Hc)
        out[f"{name}_codes"] = np.asarray(t.codes, dtype=np.uint8)
        out[f"{name}_scales"] = np.asarray(t.scale_codes, dtype=np.uint8)
        out[f"{name}_ts"] = np.float64(t.tensor_scale)
        out[f"{name}_k"] = np.int64(tr.block if tr is not None else 0)
        out[f"{name}_mse_rel"] = np.float64(res.mse_rel)
        out[f"{name}_proxy_loss"] = np.float64(loss)
        print(f"{name}: {time.time() - t0:.1f} s  proxy_loss={loss:.10g} mse_rel={res.mse_rel:.6g}", flush=True)
    np.savez_compressed(os.path.join(HERE, "gptq_fixtures.npz"), **out)


if __name__ == "__main__":
    main()
