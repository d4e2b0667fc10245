"""Drop-in exactness for the reference's other quantize_rtn inputs:

* float64 input -- the reference's own dtype (quantizers.py:96).  The GPU's float64 path
  reproduces the reference's golden container SHA-256 for the float64 Laplace blocks of
  pkg/tests/test_acceptance.py:335-361 (NVFP4 and NVFP4 + H16) and the reference's outputs on
  float64 fixtures (tests/golden/make_f64.py) for every Hadamard block.  k in {0, 16}: bit-exact
  by construction (exact products, the reference's summation order); k in {32, 64, 128}: the
  reference's own fp64 rotation depends on the BLAS kernel its shape selects, so the bar is the
  north star's >= 99.99% identical codes.
* ``ScalePolicy(e8m0_four_thirds=False)`` (quantizers.py:206-207): MXFP4 tensor scale 1.0, on
  the fast bf16 K1 path and the float64 path, bit-exact.
* NVFP4 with a static (given) global scale s_T:
  prepare_scales' arithmetic with that s_global, bit-exact against the oracle, including
  saturating groups.
"""

import hashlib
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2509_23202_b200 as P

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SPEC = {"mxfp4": P.FormatSpec.mxfp4(), "nvfp4": P.FormatSpec.nvfp4()}
GOLDEN_QUANT_SHA = {   # pkg/tests/test_acceptance.py:337-341
    "sha_nvfp4": "4b29d277a4cda8a496de9812023ea5049ab420fb2f71f4b1ddd304913e95eba1",
    "sha_hadamard": "d405df5f859ac1e05e64503c43f4b10d9198b000f8e96aea2ab8a44bd4f6d2c4",
}


@pytest.fixture(scope="module")
def f64():
    return np.load(os.path.join(HERE, "golden", "f64_fixtures.npz"))


def f64_input(seed, rows, cols, spread):   # tests/golden/make_f64.py
    rng = np.random.default_rng(int(seed))
    return rng.laplace(size=(int(rows), int(cols))) * np.exp(rng.uniform(-spread, spread, size=(int(rows), 1)))


def case_names(z):
    return sorted({k[: -len("_codes")] for k in z.files if k.endswith("_codes")})


def run_case(z, name):
    X = z["sha_x"] if name.startswith("sha_") else f64_input(*z[f"{name}_seed"])
    fmt, k = str(z[f"{name}_fmt"]), int(z[f"{name}_k"])
    pol = None if bool(z[f"{name}_four_thirds"]) else P.ScalePolicy(e8m0_four_thirds=False)
    r = P.quantize_rtn(torch.from_numpy(X).cuda(), SPEC[fmt], policy=pol,
                       transform=P.TransformSpec.hadamard(k) if k else None)
    return r, fmt, k


def test_f64_fixture_names(f64):
    assert len(case_names(f64)) == 25


@pytest.mark.parametrize("idx", range(25))
def test_float64_input_matches_reference(f64, idx):
    name = case_names(f64)[idx]
    r, fmt, k = run_case(f64, name)
    t = r.to_mfp()
    codes, scales = np.asarray(t.codes), np.asarray(t.scale_codes)
    ref_codes, ref_scales = f64[f"{name}_codes"], f64[f"{name}_scales"]
    ec = O.unpack_nibbles(codes, t.rows * t.cols)
    rc = O.unpack_nibbles(ref_codes, t.rows * t.cols)
    if k in (0, 16):
        assert np.array_equal(codes, ref_codes), (name, int((ec != rc).sum()))
        assert np.array_equal(scales, ref_scales)
        assert t.tensor_scale == float(f64[f"{name}_ts"])
    else:
        assert (ec == rc).mean() >= 0.9999, (name, int((ec != rc).sum()))
        assert (scales == ref_scales).mean() >= 0.9999
        assert t.tensor_scale == pytest.approx(float(f64[f"{name}_ts"]), rel=2 ** -22)
    m_ref = f64[f"{name}_metrics"]
    assert r.mse_rel == pytest.approx(m_ref[0], rel=1e-6)
    assert r.mse_top_rel == pytest.approx(m_ref[1], rel=1e-6, abs=1e-12)


@pytest.mark.parametrize("name", sorted(GOLDEN_QUANT_SHA))
def test_float64_reproduces_reference_golden_sha(f64, name):
    """The reference's own golden hashes, from its own float64 input, through the GPU."""
    r, _, _ = run_case(f64, name)
    blob = P.quant_bytes(r.to_mfp())
    assert hashlib.sha256(blob).hexdigest() == GOLDEN_QUANT_SHA[name]


def test_float64_nonfinite_raises():
    X = np.ones((4, 64))
    X[2, 5] = np.nan
    with pytest.raises(P.DataError, match="non-finite"):
        P.quantize_rtn(torch.from_numpy(X).cuda(), SPEC["nvfp4"])


@pytest.mark.parametrize("k", [0, 16, 32, 128])
@pytest.mark.parametrize("M,K", [(64, 1024), (300, 4096), (1, 2048)])
def test_mxfp4_without_four_thirds_bf16(M, K, k):
    rng = np.random.default_rng(M + K + k)
    X = O.bf16_round(rng.standard_normal((M, K)) * np.exp(rng.uniform(-4, 4, size=(M, 1))))
    pol = P.ScalePolicy(e8m0_four_thirds=False)
    r = P.quantize_rtn(torch.from_numpy(X).cuda().bfloat16(), SPEC["mxfp4"], policy=pol,
                       transform=P.TransformSpec.hadamard(k) if k else None)
    ora = O.quantize_rtn(X, "mxfp4", hadamard=k or None, four_thirds=False)
    assert r.tensor_scale == 1.0 == ora.tensor_scale
    ec = O.unpack_nibbles(r.codes.cpu().numpy(), M * K).reshape(M, K)
    assert np.array_equal(ec, ora.element_codes)
    assert np.array_equal(r.scale_codes().cpu().numpy(), ora.scale_codes)
    # fp32 input takes the butterfly kernel
    r32 = P.quantize_rtn(torch.from_numpy(X).cuda().float(), SPEC["mxfp4"], policy=pol,
                         transform=P.TransformSpec.hadamard(k) if k else None)
    assert torch.equal(r32.codes, r.codes) and torch.equal(r32.sf, r.sf)


@pytest.mark.parametrize("scale_mult", [0.3, 1.0, 4.0])
@pytest.mark.parametrize("k", [0, 16, 128])
@pytest.mark.parametrize("M,K", [(64, 1024), (257, 4096), (16, 4096)])
def test_nvfp4_static_tensor_scale(M, K, k, scale_mult):
    """A given s_T (e.g. calibrated offline): scale codes E4M3(raw / s_T) saturating at 448 and
    elements saturating at +-6 where the group outgrows it (scale_mult < 1)."""
    rng = np.random.default_rng(M * 3 + K + k)
    X = O.bf16_round(rng.standard_normal((M, K)))
    dyn = O.quantize_rtn(X, "nvfp4", hadamard=k or None)
    st = float(np.float32(dyn.tensor_scale * scale_mult))
    ora = O.quantize_rtn(X, "nvfp4", hadamard=k or None, static_ts=st)
    tr = P.TransformSpec.hadamard(k) if k else None
    for xt in (torch.from_numpy(X).cuda().bfloat16(), torch.from_numpy(X).cuda().float()):
        r = P.quantize_rtn(xt, SPEC["nvfp4"], transform=tr, static_tensor_scale=st)
        assert r.tensor_scale == st
        ec = O.unpack_nibbles(r.codes.cpu().numpy(), M * K).reshape(M, K)
        assert np.array_equal(ec, ora.element_codes)
        assert np.array_equal(r.scale_codes().cpu().numpy(), ora.scale_codes)
    if scale_mult == 1.0:   # s_T equal to the dynamic one: identical to the two-phase kernel
        rd = P.quantize_rtn(torch.from_numpy(X).cuda().bfloat16(), SPEC["nvfp4"], transform=tr)
        assert torch.equal(rd.codes, r.codes) and torch.equal(rd.sf, r.sf)


def test_static_tensor_scale_rejected_for_mxfp4():
    with pytest.raises(P.DataError):
        P.quantize_rtn(torch.ones((4, 64), device="cuda"), SPEC["mxfp4"], static_tensor_scale=1.0)
