"""Generate golden fixtures by running the REAL reference (microfp) in the dev container.

Usage (dev container only; /root/reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/reference_fixtures.npz``.  Every array in it is an output
of the unmodified reference API:

* ``quantize_rtn`` (pkg/src/microfp/quantizers.py:247-255) on bf16-representable
  normal / Laplace inputs for MXFP4 / NVFP4 x Hadamard k in {none,16,32,64,128},
* the edge cases SURVEY.md section 8(c) lists (zeros, on-grid blocks, exact
  ties, negative values rounding to zero, huge dynamic range),
* ``e8m0_encode`` / ``fp_scale_encode(e4m3)`` on values straddling every
  rounding threshold (formats.py:220-251),
* ``dequantize(A) @ dequantize(W).T`` in float32 (formats.py:424-442),
* the inputs of the reference's golden-hash test (test_acceptance.py:349).
"""

from __future__ import annotations

import os
import sys

import numpy as np

from microfp import (  # noqa: E402  (reference package)
    DataError, FormatSpec, ScaleFormat, TransformSpec, dequantize, e8m0_encode,
    fp_scale_encode, quantize_rtn,
)
from microfp.analysis import Sampler, sample_blocks

HERE = os.path.dirname(os.path.abspath(__file__))
SPECS = {"mxfp4": FormatSpec.mxfp4(), "nvfp4": FormatSpec.nvfp4()}
KS = [0, 16, 32, 64, 128]


def bf16(x):
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).reshape(f.shape)


def run(X, fmt, k):
    tr = TransformSpec.hadamard(k) if k else None
    r = quantize_rtn(X.astype(np.float64), SPECS[fmt], transform=tr)
    t = r.tensor
    return (np.asarray(t.codes, np.uint8).reshape(t.rows, -1),
            np.asarray(t.scale_codes, np.uint8).reshape(t.rows, -1),
            np.float64(t.tensor_scale), np.float64(r.mse_rel), np.float64(r.mse_top_rel))


def main():
    out = {}
    rng = np.random.default_rng(20250923)
    # 1. random bf16 inputs, every (format, k) combination, two distributions
    for dist in ("normal", "laplace"):
        for fmt in SPECS:
            for k in KS:
                rows, cols = 24, 512
                if dist == "normal":
                    X = rng.standard_normal((rows, cols)) * np.exp2(rng.integers(-6, 7, (rows, 1)))
                else:
                    X = rng.laplace(size=(rows, cols)) * 3.0
                X = bf16(X)
                key = f"rand_{dist}_{fmt}_k{k}"
                out[key + "_x"] = X
                (out[key + "_codes"], out[key + "_scales"], out[key + "_ts"],
                 out[key + "_mse"], out[key + "_msetop"]) = run(X, fmt, k)
    # 2. edge cases
    on_grid = np.array([6.0, 3.0, -1.5, 0.5] + [0.0] * 12)        # test_quantizers.py:33
    ties = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, -0.25,
                     -0.75, -1.25, -1.75, -2.5, -3.5, -5.0, 6.0, -6.0])
    edges = {
        "zeros": np.zeros((4, 128)),
        "ongrid": np.tile(np.concatenate([on_grid, 2 * on_grid]), (4, 4)),
        "ties": np.tile(ties, (8, 8)),
        "negsmall": np.tile(np.array([-0.01, 0.01, -0.0, 6.0] * 8), (4, 4)),
        "range": bf16(np.exp2(np.linspace(-30, 30, 8 * 128)).reshape(8, 128)
                      * np.where(np.arange(1024).reshape(8, 128) % 3 == 0, -1, 1)),
        "range12": bf16(np.exp2(np.linspace(-12, 12, 8 * 128)).reshape(8, 128)
                        * np.where(np.arange(1024).reshape(8, 128) % 5 == 0, -1, 1)),
        "zerogroup": np.concatenate([np.zeros((4, 64)), np.ones((4, 64)) * 1.5], axis=1),
    }
    for name, X in edges.items():
        X = bf16(X)
        for fmt in SPECS:
            for k in (0, 16, 32):
                key = f"edge_{name}_{fmt}_k{k}"
                out[key + "_x"] = X
                try:
                    (out[key + "_codes"], out[key + "_scales"], out[key + "_ts"],
                     out[key + "_mse"], out[key + "_msetop"]) = run(X, fmt, k)
                    out[key + "_raises"] = np.array(0)
                except DataError:
                    out[key + "_raises"] = np.array(1)
    # NVFP4 E4M3-underflow group -> the reference raises DataError (formats.py:101-102)
    X = bf16(np.concatenate([np.full((1, 16), 1e-6), np.full((1, 16), 1e6)], axis=1))
    try:
        run(X, "nvfp4", 0)
        out["err_underflow_raises"] = np.array(0)
    except DataError:
        out["err_underflow_raises"] = np.array(1)
    out["err_underflow_x"] = X
    # 3. scale-codec thresholds
    e = np.arange(-126, 127, dtype=np.float64)
    thr = np.sqrt(2.0) * np.exp2(e)
    probes = np.concatenate([thr * (1 - 2.0 ** -52), thr, thr * (1 + 2.0 ** -52),
                             np.nextafter(thr, 0), np.nextafter(thr, np.inf),
                             np.exp2(rng.uniform(-140, 140, 4000))])
    out["e8m0_in"] = probes
    out["e8m0_out"] = np.asarray(e8m0_encode(probes), np.uint8)
    lv = ScaleFormat.e4m3().levels()[:-1]
    mids = (lv[1:] + lv[:-1]) / 2
    p4 = np.concatenate([mids, np.nextafter(mids, 0), np.nextafter(mids, np.inf), lv[1:],
                         np.exp2(rng.uniform(-14, 10, 4000)), [448.0, 464.0, 500.0, 1e9]])
    out["e4m3_in"] = p4
    out["e4m3_out"] = np.asarray(fp_scale_encode(p4, ScaleFormat.e4m3()), np.uint8)
    # 4. the quantized linear (dequantize @ dequantize.T in fp32)
    for fmt in SPECS:
        for k in (0, 16, 32, 128):
            A = bf16(rng.standard_normal((16, 512)))
            W = bf16(rng.standard_normal((64, 512)) / np.sqrt(512))
            tr = TransformSpec.hadamard(k) if k else None
            ra = quantize_rtn(A.astype(np.float64), SPECS[fmt], transform=tr)
            rw = quantize_rtn(W.astype(np.float64), SPECS[fmt], transform=tr)
            Y = dequantize(ra.tensor).astype(np.float32) @ dequantize(rw.tensor).astype(np.float32).T
            key = f"lin_{fmt}_k{k}"
            out[key + "_a"], out[key + "_w"], out[key + "_y"] = A, W, Y
    # 5. inputs of the reference golden-hash test (test_acceptance.py:349)
    out["sha_x"] = sample_blocks(Sampler("laplace", 42), 64, 4)
    path = os.path.join(HERE, "reference_fixtures.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    sys.exit(main())
