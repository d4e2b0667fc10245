"""CPU-side checks of the C ABI: the library loads, exports every symbol include/mrfp4.h
declares, and rejects bad arguments synchronously (no CUDA call is reached)."""

import ctypes
import os
import re

import pytest

from paper_2509_23202_b200 import _lib
from paper_2509_23202_b200.errors import DataError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "mrfp4.h")).read()
    return sorted(set(re.findall(r"\b(mrfp4_[a-z0-9_]+)\s*\(", text)))


def test_header_and_bindings_agree():
    assert header_symbols() == sorted(_lib.SIGNATURES)


def test_library_exports_every_symbol():
    L = _lib.lib()
    for name in header_symbols():
        assert hasattr(L, name), name
    assert L.mrfp4_abi_version() == 3


def test_gemm_workspace_sizes():
    L = _lib.lib()
    assert L.mrfp4_gemm_workspace(2048, 4096, 14336, 0) == 0          # 2-CTA path: no split
    ws = L.mrfp4_gemm_workspace(16, 4096, 4096, 1)                     # C0 decode shape: split-K
    assert ws > 4096 and (ws - 4096) % (16 * 4096 * 4) == 0   # counter header + partials
    assert L.mrfp4_gemm_workspace(16, 4096, 4096, 9) == 0             # unknown format


def test_sizes():
    L = _lib.lib()
    assert L.mrfp4_group_size(0) == 32 and L.mrfp4_group_size(1) == 16 and L.mrfp4_group_size(7) == 0
    assert L.mrfp4_sf_bytes(1, 1) == 512
    assert L.mrfp4_sf_bytes(129, 5) == 256 * 8
    assert L.mrfp4_sf_bytes(2048, 448) == 2048 * 448
    assert L.mrfp4_act_quant_workspace(16, 4096, 1) == 16
    assert L.mrfp4_act_quant_workspace(2048, 14336, 0) == 0


@pytest.mark.parametrize("args,msg", [
    (dict(M=0), "non-empty"),
    (dict(K=33), "divisible by group size"),
    (dict(had_k=48), "unsupported Hadamard"),
    (dict(K=96, had_k=64), "transform block"),
    (dict(fmt=5), "unknown format"),
    (dict(x_dtype=9), "dtype"),
])
def test_act_quant_argument_errors(args, msg):
    L = _lib.lib()
    p = dict(x=16, x_dtype=0, M=4, K=64, ldx=None, fmt=0, had_k=0)
    p.update(args)
    ldx = p["ldx"] or p["K"]
    rc = L.mrfp4_act_quant(p["x"], p["x_dtype"], p["M"], p["K"], ldx, p["fmt"], p["had_k"],
                           16, 16, 16, 16, 16, 16, None)
    assert rc in (_lib.EINVAL, _lib.EUNSUPPORTED)
    assert msg in L.mrfp4_last_error().decode()
    with pytest.raises(DataError):
        _lib.check(rc)


def test_gemm_argument_errors():
    L = _lib.lib()
    rc = L.mrfp4_gemm(16, 16, 16, 16, 16, 16, 16, 0, 128, 256, 96, 256, 0, None, 0, None)
    assert rc == _lib.EUNSUPPORTED and "multiple of 64" in L.mrfp4_last_error().decode()
    rc = L.mrfp4_gemm(16, 16, 16, 16, 16, 16, 16, 0, 128, 250, 128, 256, 0, None, 0, None)
    assert rc == _lib.EUNSUPPORTED and "multiple of 8" in L.mrfp4_last_error().decode()
    rc = L.mrfp4_gemm(16, 16, 16, 16, 16, 16, 16, 5, 128, 256, 128, 256, 0, None, 0, None)
    assert rc == _lib.EUNSUPPORTED


def test_no_cuda_path_is_loud():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2509_23202_b200 as P
    with pytest.raises(RuntimeError, match="CUDA"):
        P.quantize_rtn(np.zeros((2, 32)), P.FormatSpec.mxfp4())


def test_mse_entry_points_reject_bad_arguments():
    L = _lib.lib()
    nul = None
    assert L.mrfp4_mse_pass(nul, 10, 9, nul, 129, nul, 1.0, 1.0, nul, nul, nul, nul, nul, nul) == _lib.EUNSUPPORTED
    assert L.mrfp4_mse_pass(nul, 0, 1, nul, 129, nul, 1.0, 1.0, nul, nul, nul, nul, nul, nul) == _lib.EINVAL
    assert L.mrfp4_mse_pass(nul, 10, 1, nul, 129, nul, 0.0, 1.0, nul, nul, nul, nul, nul, nul) == _lib.EINVAL
    assert L.mrfp4_mse_pass(nul, 10, 1, nul, 129, nul, 1.0, 1.0, nul, nul, nul, nul, nul, nul) == _lib.EINVAL
    assert L.mrfp4_mse_group_err(nul, 10, 0, nul, -1.0, nul, nul, nul) == _lib.EINVAL


def test_header_is_plain_c():
    """include/mrfp4.h is a C header (no C++ in the ABI): it compiles as C99 and as C++."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    hdr = os.path.join(ROOT, "include", "mrfp4.h")
    for lang, std in (("c", "-std=c99"), ("c++", "-std=c++17")):
        r = subprocess.run(["gcc", std, "-fsyntax-only", "-Wall", "-Werror", "-x", lang, hdr],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
