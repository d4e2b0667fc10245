"""MFPQ files written by the REAL reference CLI (tests/golden/make_cli.py: ``microfp quantize``,
cli.py:112-153 -> fileio.write_quant, fileio.py:138-167) through this package's weight prep --
SURVEY.md 8(f) row f2.

CPU: every file parses (fileio.py:170-226, permutation section included) and re-serializes to
the identical bytes.  GPU: ``prepare_weight(path)`` -> ``quantized_linear`` against the oracle's
dequantize-matmul of the same container; RTN files equal the GPU RTN of the CLI's own weight
tensor; the fitted-E8M0 MR-GPTQ default (``scale_fit``) is rejected, as it has no hardware form.
"""

import os
import struct

import numpy as np
import pytest

import oracle as O
import paper_2509_23202_b200 as P

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
FILES = sorted(f[:-5] for f in os.listdir(HERE) if f.endswith(".mfpq"))


def read_mfpt(path):
    """The CLI's TensorFile (fileio.py:58-90): 'MFPT', version, dtype f32, ndim, pad, uint64 dims, f32 data."""
    blob = open(path, "rb").read()
    assert blob[:4] == b"MFPT"
    ndim = blob[6]
    dims = struct.unpack(f"<{ndim}Q", blob[8:8 + 8 * ndim])
    return np.frombuffer(blob[8 + 8 * ndim:], dtype="<f4").reshape(dims)


def oracle_of(t):
    G = t.spec.group_size
    ec = O.unpack_nibbles(np.asarray(t.codes), t.rows * t.cols).reshape(t.rows, t.cols)
    fmt = "mxfp4" if G == 32 else "nvfp4"
    return O.OracleQuant(fmt, t.rows, t.cols, G, None, ec, np.asarray(t.scale_codes, np.uint8).reshape(t.rows, -1),
                         float(t.tensor_scale), 0.0, 0.0)


def test_cli_files_present():
    assert {"rtn_nvfp4_h16", "rtn_mxfp4_h32", "mrgptq_nvfp4", "mrgptq_nvfp4_h128", "mrgptq_mxfp4_absmax",
            "mrgptq_mxfp4_fit"} <= set(FILES)


@pytest.mark.parametrize("name", FILES)
def test_cli_file_parses_and_round_trips(name):
    blob = open(os.path.join(HERE, name + ".mfpq"), "rb").read()
    t, perm = P.parse_quant(blob)
    assert P.quant_bytes(t, perm=perm) == blob
    assert (perm is not None) == name.startswith("mrgptq")          # act-order permutation section
    if perm is not None:
        assert sorted(perm.tolist()) == list(range(t.cols))
    assert (t.scale_fit is not None) == name.endswith("_fit")


@pytest.mark.gpu
@pytest.mark.parametrize("name", FILES)
def test_cli_file_feeds_the_gpu_linear(name):
    import torch
    path = os.path.join(HERE, name + ".mfpq")
    t, _ = P.read_quant(path)
    if t.scale_fit is not None:
        with pytest.raises(P.DataError, match="scale_fit"):
            P.prepare_weight(path)
        return
    w = P.prepare_weight(path)
    k = w.had_k
    fmt = "mxfp4" if w.fmt == P.FMT_MXFP4 else "nvfp4"
    rng = np.random.default_rng(len(name))
    X = O.bf16_round(rng.standard_normal((96, t.cols)))
    y = P.quantized_linear(torch.from_numpy(X).cuda().bfloat16(), w, out_dtype=torch.float32).cpu().numpy()
    ref = O.linear_reference(O.quantize_rtn(X, fmt, hadamard=k or None), oracle_of(t))
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) <= 1e-5
    if name.startswith("rtn"):   # the CLI's RTN == this package's GPU RTN of the CLI's own weight
        W = read_mfpt(os.path.join(HERE, "weight.mfpt"))
        wg = P.quantize_weight(torch.from_numpy(W.copy()).cuda(), P.FormatSpec.mxfp4() if fmt == "mxfp4" else
                               P.FormatSpec.nvfp4(), P.TransformSpec.hadamard(k))
        ec = O.unpack_nibbles(wg.codes.cpu().numpy(), t.rows * t.cols)
        ref_ec = O.unpack_nibbles(np.asarray(t.codes), t.rows * t.cols)
        assert (ec == ref_ec).mean() >= 0.9999
        if k == 16:
            assert torch.equal(wg.codes, w.codes) and torch.equal(wg.sf, w.sf)
