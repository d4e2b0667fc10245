"""Golden fixtures for the GPU MSE scale search, from the REAL reference (dev container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_mse.py

Runs ``quantize(X, spec, ScalePolicy(mode=ScaleMode.MSE), transform)`` -> ``mse_optimize_scales``
(pkg/src/microfp/quantizers.py:330-347, search :263-327) on bf16-representable inputs and writes
``tests/golden/mse_fixtures.npz``: packed codes, scale codes, tensor scale and metrics per case,
plus the inputs; a case where the reference raises DataError is recorded as ``<key>_raises``.
"""

from __future__ import annotations

import os

import numpy as np

from microfp import DataError, FormatSpec, TransformSpec
from microfp.quantizers import ScaleMode, ScalePolicy, quantize

HERE = os.path.dirname(os.path.abspath(__file__))


def bf16(x):
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).reshape(f.shape)


CASES = [  # key, fmt, k, rows, cols, dist, four_thirds
    ("nv_k0_normal", "nvfp4", 0, 64, 256, "normal", True),
    ("nv_k16_laplace", "nvfp4", 16, 64, 512, "laplace", True),
    ("nv_k128_normal", "nvfp4", 128, 32, 1024, "normal", True),
    ("mx_k32_normal", "mxfp4", 32, 64, 512, "normal", True),
    ("mx_k0_laplace", "mxfp4", 0, 48, 256, "laplace", True),
    ("mx_k32_no43", "mxfp4", 32, 32, 512, "normal", False),
    ("nv_k16_scaled_rows", "nvfp4", 16, 40, 512, "rows", True),
]


def main():
    out = {}
    rng = np.random.default_rng(20251017)
    for key, fmt, k, rows, cols, dist, ft in CASES:
        if dist == "normal":
            X = rng.standard_normal((rows, cols))
        elif dist == "laplace":
            X = rng.laplace(size=(rows, cols))
        else:
            X = rng.standard_normal((rows, cols)) * np.exp2(rng.integers(-4, 5, (rows, 1)))
        X = bf16(X).astype(np.float64)
        spec = FormatSpec.mxfp4() if fmt == "mxfp4" else FormatSpec.nvfp4()
        pol = ScalePolicy(mode=ScaleMode.MSE, e8m0_four_thirds=ft)
        r = quantize(X, spec, policy=pol, transform=TransformSpec.hadamard(k) if k else None)
        t = r.tensor
        out[key + "_x"] = X.astype(np.float32)
        out[key + "_codes"] = np.asarray(t.codes, np.uint8).reshape(rows, -1)
        out[key + "_scales"] = np.asarray(t.scale_codes, np.uint8).reshape(rows, -1)
        out[key + "_ts"] = np.float64(t.tensor_scale)
        out[key + "_mse"] = np.array([r.mse_rel, r.mse_top_rel])
        print(key, t.tensor_scale, r.mse_rel)
    # NVFP4 tiny groups next to a huge one: the 0.5x candidate underflows E4M3 -> DataError
    X = bf16(rng.standard_normal((8, 256)) * 1e-3).astype(np.float64)
    X[0, 0] = 3.0e4
    try:
        quantize(X, FormatSpec.nvfp4(), policy=ScalePolicy(mode=ScaleMode.MSE))
        raises = False
    except DataError:
        raises = True
    out["nv_underflow_x"] = X.astype(np.float32)
    out["nv_underflow_raises"] = np.bool_(raises)
    print("underflow raises:", raises)
    np.savez_compressed(os.path.join(HERE, "mse_fixtures.npz"), **out)


if __name__ == "__main__":
    main()
