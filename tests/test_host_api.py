"""Host-side API mirror: format/transform mapping, container invariants, MFPQ I/O."""

import hashlib
import os
import sys

import numpy as np
import pytest

import oracle as O
import paper_2509_23202_b200 as P
from paper_2509_23202_b200.formats import format_code
from paper_2509_23202_b200.transforms import hadamard_block


def test_format_codes():
    assert format_code(P.FormatSpec.mxfp4()) == P.FMT_MXFP4
    assert format_code(P.FormatSpec.nvfp4()) == P.FMT_NVFP4
    for bad in (P.FormatSpec(16, P.ScaleFormat.e8m0()), P.FormatSpec(32, P.ScaleFormat.e4m3()),
                P.FormatSpec(16, P.ScaleFormat.e4m3(), global_scale=False),
                P.FormatSpec(16, P.ScaleFormat.unquantized()), P.FormatSpec(16, P.ScaleFormat.fpem(3, 4), True)):
        with pytest.raises(P.DataError, match="unsupported"):
            format_code(bad)


def test_transform_mapping():
    assert hadamard_block(None) == 0
    assert hadamard_block(P.TransformSpec.identity(16)) == 0
    for k in (16, 32, 64, 128):
        assert hadamard_block(P.TransformSpec.hadamard(k)) == k
    with pytest.raises(P.DataError):
        hadamard_block(P.TransformSpec.hadamard(256))
    with pytest.raises(P.DataError):
        hadamard_block(P.TransformSpec(P.TransformKind.DCT2, 16))
    with pytest.raises(P.DataError):
        P.TransformSpec.hadamard(24)


def test_reference_objects_are_accepted_when_available():
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present (GPU box)")
    sys.path.insert(0, ref)
    try:
        import microfp
        assert format_code(microfp.FormatSpec.mxfp4()) == P.FMT_MXFP4
        assert format_code(microfp.FormatSpec.nvfp4()) == P.FMT_NVFP4
        assert hadamard_block(microfp.TransformSpec.hadamard(128)) == 128
    finally:
        sys.path.remove(ref)


def test_container_invariants():
    spec = P.FormatSpec.mxfp4()
    with pytest.raises(P.DataError, match="reserved"):
        P.pack_tensor(np.zeros((1, 32), np.uint8), np.array([255], np.uint8), spec)
    with pytest.raises(P.DataError):
        P.pack_tensor(np.zeros((1, 33), np.uint8), np.array([127], np.uint8), spec, dims=(1, 33))
    t = P.pack_tensor(np.array([[1, 2] + [0] * 30]), np.array([127]), spec)
    assert t.codes[0] == 1 | (2 << 4)
    ec, sc = P.unpack_tensor(t)
    assert ec[0, 0] == 1 and ec[0, 1] == 2 and sc[0] == 127


def test_mfpq_writer_reproduces_reference_golden_hash(golden):
    """quant_bytes of the oracle result == the reference's golden SHA (test_acceptance.py:337-339)."""
    X = golden["sha_x"]
    q = O.quantize_rtn(X, O.NVFP4, hadamard=16)
    t = P.MfpTensor(P.FormatSpec.nvfp4(), q.rows, q.cols, q.codes.reshape(-1), q.scale_codes.reshape(-1),
                    q.tensor_scale, P.TransformSpec.hadamard(16), None)
    blob = P.quant_bytes(t)
    assert hashlib.sha256(blob).hexdigest() == "d405df5f859ac1e05e64503c43f4b10d9198b000f8e96aea2ab8a44bd4f6d2c4"
    t2, perm = P.parse_quant(blob)
    assert perm is None and t2.rows == t.rows and t2.tensor_scale == t.tensor_scale
    np.testing.assert_array_equal(t2.codes, t.codes)
    np.testing.assert_array_equal(t2.scale_codes, t.scale_codes)
    assert t2.transform == P.TransformSpec.hadamard(16)


def test_mfpq_errors(tmp_path):
    with pytest.raises(P.DataError, match="not a QuantFile"):
        P.parse_quant(b"XXXX\x01\x00\x00\x00\x00")
    q = O.quantize_rtn(np.ones((2, 32)), O.MXFP4)
    t = P.MfpTensor(P.FormatSpec.mxfp4(), 2, 32, q.codes.reshape(-1), q.scale_codes.reshape(-1), q.tensor_scale)
    blob = P.quant_bytes(t, perm=np.arange(32))
    t2, perm = P.parse_quant(blob)
    np.testing.assert_array_equal(perm, np.arange(32))
    with pytest.raises(P.DataError, match="size mismatch"):
        P.parse_quant(blob[:-1])
    path = tmp_path / "w.mfpq"
    P.write_quant(path, t)
    t3, _ = P.read_quant(path)
    assert t3.rows == 2
