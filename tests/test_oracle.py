"""Pin the CPU oracle against the real reference (fixtures + golden hashes + known answers).

Fixtures: ``tests/golden/reference_fixtures.npz`` written by
``tests/golden/make_golden.py`` from the unmodified reference package.
Known answers restate the reference's own unit tests (pkg/tests/test_formats.py,
pkg/tests/test_quantizers.py); golden hashes are test_acceptance.py:335-361.
"""

import hashlib

import numpy as np
import pytest

import oracle as O

GOLDEN_QUANT_SHA = {  # pkg/tests/test_acceptance.py:336-340
    "nvfp4": "4b29d277a4cda8a496de9812023ea5049ab420fb2f71f4b1ddd304913e95eba1",
    "hadamard": "d405df5f859ac1e05e64503c43f4b10d9198b000f8e96aea2ab8a44bd4f6d2c4",
}


def test_golden_container_hashes(golden):
    X = golden["sha_x"]
    got = {
        "nvfp4": O.mfpq_bytes(O.quantize_rtn(X, O.NVFP4)),
        "hadamard": O.mfpq_bytes(O.quantize_rtn(X, O.NVFP4, hadamard=16)),
    }
    for name, blob in got.items():
        assert hashlib.sha256(blob).hexdigest() == GOLDEN_QUANT_SHA[name], name


def _keys(golden, prefix):
    return sorted({k[: -len("_x")] for k in golden.files if k.startswith(prefix) and k.endswith("_x")})


def _check(golden, key):
    X = golden[key + "_x"]
    parts = key.split("_")
    fmt, k = parts[-2], int(parts[-1][1:])
    raises = key + "_raises" in golden.files and int(golden[key + "_raises"])
    if raises:
        with pytest.raises(O.OracleDataError):
            O.quantize_rtn(X, fmt, hadamard=k or None)
        return
    q = O.quantize_rtn(X, fmt, hadamard=k or None)
    np.testing.assert_array_equal(q.codes, golden[key + "_codes"])
    np.testing.assert_array_equal(q.scale_codes, golden[key + "_scales"])
    assert q.tensor_scale == float(golden[key + "_ts"])
    assert q.mse_rel == pytest.approx(float(golden[key + "_mse"]), rel=1e-9, abs=1e-300)
    assert q.mse_top_rel == pytest.approx(float(golden[key + "_msetop"]), rel=1e-9, abs=1e-300)


def test_random_fixtures_bit_exact(golden):
    keys = _keys(golden, "rand_")
    assert len(keys) == 20
    for key in keys:
        _check(golden, key)


def test_edge_fixtures_bit_exact(golden):
    keys = _keys(golden, "edge_")
    assert len(keys) >= 36
    for key in keys:
        _check(golden, key)


def test_underflow_raises(golden):
    assert int(golden["err_underflow_raises"]) == 1
    with pytest.raises(O.OracleDataError):
        O.quantize_rtn(golden["err_underflow_x"], O.NVFP4)


def test_scale_codecs_match_reference(golden):
    np.testing.assert_array_equal(O.e8m0_encode(golden["e8m0_in"]), golden["e8m0_out"])
    np.testing.assert_array_equal(O.e4m3_encode(golden["e4m3_in"]), golden["e4m3_out"])


def test_linear_fixtures(golden):
    for fmt in ("mxfp4", "nvfp4"):
        for k in (0, 16, 32, 128):
            key = f"lin_{fmt}_k{k}"
            A = O.quantize_rtn(golden[key + "_a"], fmt, hadamard=k or None)
            W = O.quantize_rtn(golden[key + "_w"], fmt, hadamard=k or None)
            np.testing.assert_array_equal(O.linear_reference(A, W), golden[key + "_y"])


# ---- known answers restated from the reference's unit tests -----------------

@pytest.mark.parametrize("x,expected", [            # test_formats.py:39-52
    (0.24, 0.0), (7.3, 6.0), (-1.3, -1.5), (2.5, 2.0), (0.25, 0.0), (0.75, 1.0),
    (1.25, 1.0), (1.75, 2.0), (3.5, 4.0), (5.0, 4.0), (-2.5, -2.0), (0.0, 0.0)])
def test_fp4_examples(x, expected):
    c = O.fp4_codes(np.array([x]))
    v = O.FP4_GRID[c & 7] * np.where(c & 8, -1, 1)
    assert float(v[0]) == expected


def test_fp4_negative_zero_canonical():            # formats.py:110, test_formats.py:96-101
    np.testing.assert_array_equal(O.fp4_codes(np.array([-0.1, -0.0, 0.1, -0.25])), [0, 0, 0, 0])


def test_e8m0_known_answers():                     # test_formats.py:108-142
    assert O.e8m0_encode(1.0) == 127
    assert O.e8m0_encode(0.8333) == 127
    assert O.e8m0_encode(1e300) == 254 and O.e8m0_encode(1e-300) == 0
    np.testing.assert_array_equal(O.e8m0_encode(np.ldexp(1.0, np.arange(255) - 127)), np.arange(255))


def test_e4m3_known_answers():                     # test_formats.py:150-206
    assert O.E4M3_LEVELS[126] == 448.0 and O.E4M3_LEVELS[1] == 2.0 ** -9
    np.testing.assert_array_equal(O.e4m3_encode(O.E4M3_LEVELS[1:]), np.arange(1, 127))
    assert O.e4m3_encode(500.0) == 126 and O.e4m3_encode(1e30) == 126
    mids = (O.E4M3_LEVELS[1:] + O.E4M3_LEVELS[:-1]) / 2
    assert (O.e4m3_encode(mids[1:]) % 2 == 0).all()


def test_mxfp4_four_thirds():                      # test_quantizers.py:62-71
    X = np.concatenate([[5.0], np.zeros(31)])[None, :]
    q = O.quantize_rtn(X, O.MXFP4)
    assert q.scale_codes[0, 0] == 127
    assert q.tensor_scale == float(np.float32(4 / 3))


def test_nvfp4_global_scale_top_is_448():          # test_quantizers.py:83-90
    X = np.random.default_rng(0).laplace(scale=200.0, size=(16, 64))
    q = O.quantize_rtn(X, O.NVFP4)
    assert O.E4M3_LEVELS[q.scale_codes].max() == 448.0


def test_zero_sentinels():                          # SURVEY.md 8(c) edge fixtures
    q = O.quantize_rtn(np.zeros((2, 64)), O.NVFP4)
    assert (q.scale_codes == 56).all() and q.tensor_scale == 1.0
    q = O.quantize_rtn(np.zeros((2, 64)), O.MXFP4)
    assert (q.scale_codes == 127).all()


def test_hadamard_orthogonal():                     # test_transforms.py:33-38
    for k in (2, 16, 32, 64, 128, 256):
        U = O.hadamard_matrix(k)
        np.testing.assert_allclose(U @ U.T, np.eye(k), atol=1e-12)


def test_packing_low_nibble_first():               # test_formats.py:251-255
    assert O.pack_nibbles(np.array([1, 2], np.uint8))[0] == 1 | (2 << 4)


def test_sf_swizzle_roundtrip_and_formula():
    rng = np.random.default_rng(5)
    for rows, cols in [(1, 1), (128, 4), (130, 7), (300, 33)]:
        sf = rng.integers(0, 255, (rows, cols), dtype=np.uint8)
        buf = O.sf_swizzle(sf)
        assert buf.size == O.sf_swizzled_size(rows, cols)
        np.testing.assert_array_equal(O.sf_unswizzle(buf, rows, cols), sf)
    # spot-check the 128x4 atom: row r, col c -> (r%32)*16 + (r//32)*4 + c
    sf = np.arange(128 * 4, dtype=np.int64).reshape(128, 4).astype(np.uint8)
    buf = O.sf_swizzle(sf)
    for r in (0, 1, 31, 32, 33, 127):
        for c in range(4):
            assert buf[(r % 32) * 16 + (r // 32) * 4 + c] == sf[r, c]
