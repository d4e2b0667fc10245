"""ctypes binding of libmrfp4.so (the C ABI declared in include/mrfp4.h).

The library is built in-tree by ``make`` (``__graft_entry__.build()``).  There is
no fallback: if the shared object is missing or CUDA is unavailable, every GPU
entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DataError

_HERE = os.path.dirname(os.path.abspath(__file__))
# MRFP4_LIB: an alternative build of the same library (perf experiments, e.g. the MRFP4_TRACE build)
LIB_PATH = os.environ.get("MRFP4_LIB") or os.path.join(_HERE, "libmrfp4.so")

OK, EINVAL, EUNSUPPORTED, ECUDA = 0, 1, 2, 3
DT_BF16, DT_F16, DT_F32, DT_F64 = 0, 1, 2, 3
STATUS_NONFINITE, STATUS_SCALE_UNDERFLOW = 1, 2

_lock = threading.Lock()
_lib = None

_c = ctypes
_vp, _i64, _int, _sz = _c.c_void_p, _c.c_int64, _c.c_int, _c.c_size_t


class ActQuantOpts(ctypes.Structure):
    """mrfp4_act_quant_opts (include/mrfp4.h)."""
    _fields_ = [("mx_four_thirds", ctypes.c_int), ("nv_tensor_scale", ctypes.c_void_p)]
SIGNATURES = {
    "mrfp4_abi_version": (_int, []),
    "mrfp4_last_error": (_c.c_char_p, []),
    "mrfp4_group_size": (_int, [_int]),
    "mrfp4_sf_bytes": (_sz, [_i64, _i64]),
    "mrfp4_act_quant_workspace": (_sz, [_i64, _i64, _int]),
    "mrfp4_act_quant": (_int, [_vp, _int, _i64, _i64, _i64, _int, _int, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "mrfp4_act_quant_ex": (_int, [_vp, _int, _i64, _i64, _i64, _int, _int, _vp, _vp, _vp, _vp, _vp, _sz,
                                  _c.POINTER(ActQuantOpts), _vp]),
    "mrfp4_rotate_f64": (_int, [_vp, _i64, _i64, _i64, _int, _vp, _vp]),
    "mrfp4_quant_metrics": (_int, [_vp, _int, _i64, _i64, _i64, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "mrfp4_sf_swizzle": (_int, [_vp, _vp, _i64, _i64, _vp]),
    "mrfp4_sf_unswizzle": (_int, [_vp, _vp, _i64, _i64, _vp]),
    "mrfp4_gemm_workspace": (_sz, [_i64, _i64, _i64, _int]),
    "mrfp4_gemm": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _int, _i64, _i64, _i64, _i64, _int, _vp, _sz, _vp]),
    "mrfp4_dequantize": (_int, [_vp, _vp, _vp, _i64, _i64, _int, _vp, _vp]),
    "mrfp4_gemm_quant_next": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _int, _int, _vp, _vp,
                                     _vp, _vp, _vp]),
    "mrfp4_gemm_quant_next_ex": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _int, _int, _int,
                                        _vp, _vp, _vp, _vp, _vp, _vp]),
    "mrfp4_mse_pass": (_int, [_vp, _i64, _int, _vp, _int, _vp, _c.c_double, _c.c_double, _vp, _vp, _vp, _vp, _vp,
                              _vp]),
    "mrfp4_mse_group_err": (_int, [_vp, _i64, _int, _vp, _c.c_double, _vp, _vp, _vp]),
    "mrfp4_gemm_peers": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _c.POINTER(_vp), _int, _i64, _i64, _i64, _i64, _int,
                                _vp]),
    "mrfp4_linear_decode_workspace": (_sz, [_i64, _i64, _i64]),
    "mrfp4_linear_decode_ctas": (_int, [_i64, _i64, _i64]),
    "mrfp4_linear_decode": (_int, [_vp, _int, _i64, _i64, _int, _int, _vp, _vp, _vp, _i64, _vp, _int, _i64, _vp, _sz,
                                   _vp, _vp]),
    "mrfp4_gptq_block": (_int, [_vp, _vp, _vp, _i64, _i64, _int, _int, _vp, _vp, _vp, _vp]),
    "mrfp4_pairwise_sums": (_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
}


def lib():
    """Load (once) and return the ctypes handle; raises if the library is missing."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} not found: build the CUDA extension first "
                        "(`make` or `python -c 'import __graft_entry__ as g; g.build()'`)")
                handle = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(handle, name)
                    fn.restype, fn.argtypes = res, args
                if handle.mrfp4_abi_version() != 3:
                    raise ImportError("libmrfp4.so ABI version mismatch")
                _lib = handle
    return _lib


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception convention."""
    if rc == OK:
        return
    msg = lib().mrfp4_last_error().decode(errors="replace")
    if rc in (EINVAL, EUNSUPPORTED):
        raise DataError(msg)
    raise RuntimeError(msg)


def ptr(t) -> int:
    return t.data_ptr() if t is not None else 0


def stream_ptr(torch_mod, device=None) -> int:
    return torch_mod.cuda.current_stream(device).cuda_stream
