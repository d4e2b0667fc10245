"""Generate MR-GPTQ weight fixtures by running the REAL reference (microfp) in the dev container.

Usage (dev container only; /root/reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_mrgptq.py

Writes ``tests/golden/mrgptq_fixtures.npz``: weights quantized by the unmodified reference
solver (pkg/src/microfp/gptq.py) -- the producers the north star names for the weight side
of ``Q(X H_k) Q(W H_k)^T`` -- plus the activations, their reference RTN quantization and the
reference linear output ``dequantize(Aq) @ dequantize(Wq).T`` (formats.py:424-442):

* ``mr_gptq(W, H, nvfp4)`` (gptq.py:274-300): Hadamard-16, MSE-searched E4M3 scales
  (quantizers.py:263-327), act-order; hardware-consumable (E4M3 + global scale).
* ``gptq_quantize(W, H, mxfp4, GptqConfig(act_order=True, transform=H_32, ScalePolicy()))``
  (gptq.py:181-238): the hardware-compatible MR-MXFP4 configuration (absmax + 4/3 E8M0 --
  what ``microfp quantize --method mr-gptq --scale-opt absmax`` produces, cli.py:94-109).
* ``mr_gptq(W, H, mxfp4)`` default: fitted E8M0 grid (``scale_fit``, gptq.py:293-294) --
  NOT hardware E8M0; the GPU path must reject it.

Shapes are small slices (rows x K) so the CPU solver runs in seconds.
"""

from __future__ import annotations

import os

import numpy as np

from microfp import FormatSpec, GptqConfig, ScalePolicy, TransformSpec, dequantize, quantize_rtn  # noqa: E402
from microfp.gptq import Hessian, accumulate_hessian, gptq_quantize, mr_gptq  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def bf16(x):
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def main():
    rng = np.random.default_rng(2509)
    rows, K, M = 128, 512, 64
    W = rng.standard_normal((rows, K)) / np.sqrt(K)
    Xc = rng.standard_normal((256, K))                      # calibration activations
    H = accumulate_hessian(Xc, Hessian(K))
    X = bf16(rng.standard_normal((M, K)))                   # online activations
    out = {"W": W, "X": X}
    cases = {
        "mrgptq_nvfp4_h16": (mr_gptq(W, H, FormatSpec.nvfp4()), "nvfp4", 16),
        "gptq_mxfp4_h32_absmax": (gptq_quantize(W, H, FormatSpec.mxfp4(), GptqConfig(
            act_order=True, transform=TransformSpec.hadamard(32), scale_policy=ScalePolicy())), "mxfp4", 32),
        "mrgptq_mxfp4_fit": (mr_gptq(W, H, FormatSpec.mxfp4()), "mxfp4", 32),
    }
    for name, (res, fmt, k) in cases.items():
        t = res.tensor
        out[f"{name}_codes"] = np.asarray(t.codes, dtype=np.uint8)
        out[f"{name}_scales"] = np.asarray(t.scale_codes)
        out[f"{name}_ts"] = np.float64(t.tensor_scale)
        out[f"{name}_fit"] = np.asarray(t.scale_fit if t.scale_fit is not None else (np.nan, np.nan), dtype=np.float64)
        out[f"{name}_k"] = np.int64(k)
        if t.scale_fit is None:
            spec = FormatSpec.mxfp4() if fmt == "mxfp4" else FormatSpec.nvfp4()
            Aq = quantize_rtn(X, spec, transform=TransformSpec.hadamard(k)).tensor
            out[f"{name}_y"] = (dequantize(Aq).astype(np.float32) @ dequantize(t).astype(np.float32).T)
    np.savez_compressed(os.path.join(HERE, "mrgptq_fixtures.npz"), **out)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
