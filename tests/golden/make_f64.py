"""Float64-input fixtures from the REAL reference (microfp), for the GPU's float64 path.

Usage (dev container only; /root/reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_f64.py

The reference quantizes in float64 (quantizers.py:96); its own golden container hashes
(pkg/tests/test_acceptance.py:335-361) are made from float64 Laplace blocks
``sample_blocks(Sampler("laplace", 42), 64, 4)`` that no bf16/fp32 kernel can represent.
Writes ``tests/golden/f64_fixtures.npz``: that input, the reference's quantize_rtn outputs
for NVFP4, NVFP4 + H16 and MXFP4 (4/3 and e8m0_four_thirds=False), and float64 random cases
for every Hadamard block, with the reference's codes / scale codes / tensor scale / metrics.
"""

from __future__ import annotations

import os

import numpy as np

from microfp import FormatSpec, ScalePolicy, TransformSpec, quantize_rtn  # noqa: E402
from microfp.analysis import Sampler, sample_blocks  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def f64_input(seed, rows, cols, spread):
    """Laplace rows with per-row magnitudes e^U(-spread, spread) (NVFP4 keeps spread small: its
    whole-tensor s_T must leave every group above the E4M3 underflow the reference rejects)."""
    rng = np.random.default_rng(seed)
    return rng.laplace(size=(rows, cols)) * np.exp(rng.uniform(-spread, spread, size=(rows, 1)))


def main():
    out = {}
    X = np.asarray(sample_blocks(Sampler("laplace", 42), 64, 4), dtype=np.float64)
    out["sha_x"] = X
    cases = {
        "sha_nvfp4": (X, FormatSpec.nvfp4(), None, None),
        "sha_hadamard": (X, FormatSpec.nvfp4(), None, TransformSpec.hadamard(16)),
        "sha_mxfp4": (X, FormatSpec.mxfp4(), None, None),
        "sha_mxfp4_no43": (X, FormatSpec.mxfp4(), ScalePolicy(e8m0_four_thirds=False), None),
    }
    seeds = {}
    for k in (0, 16, 32, 64, 128):
        for fmt in ("nvfp4", "mxfp4"):
            for rows, cols in ((4, 256), (32, 512)):
                name = f"r_{fmt}_k{k}_{rows}x{cols}"
                seeds[name] = (len(seeds) + 1, rows, cols, 2 if fmt == "nvfp4" else 6)
                spec = FormatSpec.nvfp4() if fmt == "nvfp4" else FormatSpec.mxfp4()
                cases[name] = (f64_input(*seeds[name]), spec, None, TransformSpec.hadamard(k) if k else None)
    seeds["r_mxfp4_no43_k32"] = (99, 32, 512, 6)
    cases["r_mxfp4_no43_k32"] = (f64_input(*seeds["r_mxfp4_no43_k32"]), FormatSpec.mxfp4(),
                                 ScalePolicy(e8m0_four_thirds=False), TransformSpec.hadamard(32))
    for name, (Xc, spec, pol, tr) in cases.items():
        r = quantize_rtn(Xc, spec, policy=pol, transform=tr)
        t = r.tensor
        if name in seeds:
            out[f"{name}_seed"] = np.array(seeds[name], dtype=np.int64)   # the test regenerates X
        out[f"{name}_fmt"] = np.array("nvfp4" if spec.group_size == 16 else "mxfp4")
        out[f"{name}_k"] = np.int64(tr.block if tr is not None else 0)
        out[f"{name}_four_thirds"] = np.bool_(pol is None or pol.e8m0_four_thirds)
        out[f"{name}_codes"] = np.asarray(t.codes, dtype=np.uint8)
        out[f"{name}_scales"] = np.asarray(t.scale_codes, dtype=np.uint8)
        out[f"{name}_ts"] = np.float64(t.tensor_scale)
        out[f"{name}_metrics"] = np.array([r.mse_rel, r.mse_top_rel], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "f64_fixtures.npz"), **out)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
