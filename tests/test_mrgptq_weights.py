"""MR-GPTQ / GPTQ weights produced by the real reference solver (gptq.py) feed the GPU path.

Fixtures: tests/golden/mrgptq_fixtures.npz, made by tests/golden/make_mrgptq.py running the
unmodified reference (``mr_gptq`` NVFP4 + Hadamard-16 with MSE scales; hardware-compatible
MR-MXFP4 = ``gptq_quantize(act_order, H_32, absmax)``; and the default ``mr_gptq`` MXFP4 with a
fitted E8M0 grid, which has no hardware encoding and must be rejected).
"""

import os

import numpy as np
import pytest

import oracle as O
import paper_2509_23202_b200 as P

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mrgptq_fixtures.npz")
CASES = {"mrgptq_nvfp4_h16": "nvfp4", "gptq_mxfp4_h32_absmax": "mxfp4"}


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def container(gold, name, fmt):
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    W = gold["W"]
    fit = gold[f"{name}_fit"]
    return P.MfpTensor(spec, W.shape[0], W.shape[1], gold[f"{name}_codes"], gold[f"{name}_scales"],
                       float(gold[f"{name}_ts"]), P.TransformSpec.hadamard(int(gold[f"{name}_k"])),
                       None if np.isnan(fit).all() else (float(fit[0]), float(fit[1])))


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_linear_matches_reference_on_gptq_weights(gold, name):
    """Pins the oracle's dequantize/linear on solver-produced weights (formats.py:424-442)."""
    fmt = CASES[name]
    t = container(gold, name, fmt)
    k = int(gold[f"{name}_k"])
    Aq = O.quantize_rtn(gold["X"], fmt, hadamard=k)
    G = t.spec.group_size
    Wq = O.OracleQuant(fmt, t.rows, t.cols, G, k, t.element_codes(), np.asarray(t.scale_codes).reshape(t.rows, -1),
                       t.tensor_scale, 0.0, 0.0)
    y = O.linear_reference(Aq, Wq).astype(np.float32)
    np.testing.assert_allclose(y, gold[f"{name}_y"], rtol=1e-6, atol=1e-6 * np.abs(gold[f"{name}_y"]).max())


def test_fitted_e8m0_weights_rejected(gold):
    """mr_gptq's default MXFP4 grid 2^(a*q+b) is not hardware E8M0."""
    t = container(gold, "mrgptq_mxfp4_fit", "mxfp4")
    assert t.scale_fit is not None
    with pytest.raises(P.DataError, match="scale_fit"):
        P.prepare_weight(t)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_gpu_linear_on_gptq_weights(gold, name):
    """prepare_weight(MfpTensor from the reference solver) + quantized_linear == reference."""
    import torch
    fmt = CASES[name]
    w = P.prepare_weight(container(gold, name, fmt))
    x = torch.from_numpy(gold["X"].astype(np.float32)).cuda().bfloat16()
    y = P.quantized_linear(x, w, out_dtype=torch.float32).cpu().numpy()
    ref = gold[f"{name}_y"]
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) <= 1e-5
