"""Numpy restatement of the reference's quantized-linear hot path (TEST INFRASTRUCTURE).

This module is the parity checker for the CUDA path in ``paper_2509_23202_b200``.
It is NOT part of the product: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU legs may use it.  It restates, in float64 numpy, the
reference functions named below (paths relative to ``/root/reference``):

* FP4 E2M1 round-to-nearest-even with the -0 -> code 0 rule
  (``pkg/src/microfp/formats.py:50-60`` grid/ties, ``:94-113`` ``fp4_round_codes``)
* E8M0 log-domain encode (``formats.py:220-227``) and E4M3 level table + RNE
  encode (``formats.py:191-210``, ``:81-91``, ``:239-251``)
* Sylvester Hadamard / sqrt(k) and the block-wise row rotation
  (``pkg/src/microfp/transforms.py:56-69``, ``:77-91``)
* absmax group scales, NVFP4 whole-tensor global scale, MXFP4 4/3 factor
  (``pkg/src/microfp/quantizers.py:170-208``), element quantization
  (``quantizers.py:211-215``), metrics (``quantizers.py:218-231``) and the
  ``quantize_rtn`` composition (``quantizers.py:247-255``)
* low-nibble-first packing (``formats.py:377-382``) and ``dequantize``
  (``formats.py:424-442``)
* the MFPQ container byte layout (``pkg/src/microfp/fileio.py:138-167``), used
  only to pin this oracle against the reference's golden SHA-256 hashes
* the tensor-core scale-factor layout (cuBLAS "blocked" 128x4 atoms; not a
  reference function -- the hardware layout the GPU path writes, SURVEY.md
  Appendix B).

Parity status: PINNED.  ``tests/test_oracle.py`` checks this module against
fixtures produced by running the real reference (``tests/golden/make_golden.py``)
and against the reference's own golden hashes.
"""

from __future__ import annotations

import dataclasses
import struct

import numpy as np

__all__ = [
    "MXFP4",
    "NVFP4",
    "OracleDataError",
    "OracleQuant",
    "FP4_GRID",
    "E4M3_LEVELS",
    "fp4_codes",
    "e8m0_encode",
    "e4m3_encode",
    "hadamard_matrix",
    "rotate_blockwise",
    "quantize_rtn",
    "dequantize",
    "linear_reference",
    "pack_nibbles",
    "unpack_nibbles",
    "sf_swizzle",
    "sf_unswizzle",
    "sf_swizzled_size",
    "mfpq_bytes",
    "bf16_round",
    "quantize_rtn_parallel",
    "dequantize_f32",
]

MXFP4 = "mxfp4"
NVFP4 = "nvfp4"


class OracleDataError(ValueError):
    """Mirror of microfp.errors.DataError (``pkg/src/microfp/errors.py:8-9``)."""


# E2M1 magnitudes indexed by the 3-bit magnitude code (formats.py:50-53).
FP4_GRID = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
# Decision points between consecutive grid values and whether an exact tie
# rounds up (to the even mantissa), formats.py:57-60.
_FP4_MIDS = (FP4_GRID[1:] + FP4_GRID[:-1]) * 0.5
_FP4_TIE_UP = np.array([False, True, False, True, False, True, False])


def _e4m3_levels() -> np.ndarray:
    """Finite E4M3 scale levels by code 0..126 (formats.py:197-205; 127 reserved)."""
    c = np.arange(127)
    e, m = c >> 3, c & 7
    sub = m * 2.0 ** -9
    norm = (1.0 + m / 8.0) * np.exp2(e - 7.0)
    return np.where(e == 0, sub, norm)


E4M3_LEVELS = _e4m3_levels()
_E4M3_MIDS = (E4M3_LEVELS[1:] + E4M3_LEVELS[:-1]) * 0.5
E4M3_MAX = float(E4M3_LEVELS[-1])  # 448
FOUR_THIRDS_F32 = float(np.float32(4.0 / 3.0))  # quantizers.py:34, :191


def fp4_codes(u) -> np.ndarray:
    """4-bit E2M1 codes of ``u`` (RNE, saturating at 6, -0 -> 0).  formats.py:94-113."""
    u = np.asarray(u, dtype=np.float64)
    if not np.isfinite(u).all():
        raise OracleDataError("non-finite element")
    mag = np.abs(u)
    idx = np.zeros(u.shape, dtype=np.uint8)
    for i, mid in enumerate(_FP4_MIDS):
        idx += (mag > mid)
        if _FP4_TIE_UP[i]:
            idx += (mag == mid)
    neg = np.signbit(u) & (idx > 0)
    return (idx | (neg.astype(np.uint8) << 3)).astype(np.uint8)


def fp4_values(codes) -> np.ndarray:
    c = np.asarray(codes, dtype=np.intp)
    v = FP4_GRID[c & 7]
    return np.where(c & 8, -v, v)


def e8m0_encode(s) -> np.ndarray:
    """clamp(rint(log2 s), -127, 127) + 127  (formats.py:220-227)."""
    s = np.asarray(s, dtype=np.float64)
    if not (np.isfinite(s).all() and (s > 0).all()):
        raise OracleDataError("E8M0 scale must be finite and positive")
    return (np.clip(np.rint(np.log2(s)), -127, 127) + 127).astype(np.uint8)


def e4m3_encode(s) -> np.ndarray:
    """RNE of positive ``s`` onto the 127 finite E4M3 levels, saturating at 448.

    formats.py:239-251 with the tie rule of ``_rtn_even`` (formats.py:81-91):
    an exact midpoint goes to the even code.
    """
    s = np.asarray(s, dtype=np.float64)
    if not (np.isfinite(s).all() and (s > 0).all()):
        raise OracleDataError("scale must be finite and positive")
    below = np.searchsorted(_E4M3_MIDS, s, side="left")  # count of mids < s
    j = np.minimum(below, _E4M3_MIDS.size - 1)
    tie_to_even = (below < _E4M3_MIDS.size) & (s == _E4M3_MIDS[j]) & (j % 2 == 1)
    return np.minimum(below + tie_to_even, 126).astype(np.uint8)


def hadamard_matrix(k: int) -> np.ndarray:
    """Sylvester-order H_k / sqrt(k)  (transforms.py:56-69)."""
    if k < 1 or k & (k - 1):
        raise OracleDataError("Hadamard block must be a power of two")
    h = np.array([[1.0]])
    while h.shape[0] < k:
        h = np.kron(np.array([[1.0, 1.0], [1.0, -1.0]]), h)
    return h / np.sqrt(k)


def rotate_blockwise(X, k: int | None) -> np.ndarray:
    """Row-vector block rotation Y_blk = X_blk @ U^T  (transforms.py:77-91)."""
    X = np.asarray(X, dtype=np.float64)
    if not k:
        return X.copy()
    rows, cols = X.shape
    if cols % k:
        raise OracleDataError(f"columns ({cols}) not divisible by transform block ({k})")
    U = hadamard_matrix(k)
    return (X.reshape(rows, cols // k, k) @ U.T).reshape(rows, cols)


def pack_nibbles(codes) -> np.ndarray:
    """Two codes per byte, earlier element in the low nibble (formats.py:377-382)."""
    flat = np.asarray(codes, dtype=np.uint8).reshape(-1)
    if flat.size % 2:
        flat = np.append(flat, np.uint8(0))
    return (flat[0::2] | (flat[1::2] << 4)).astype(np.uint8)


def unpack_nibbles(packed, n: int) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8).reshape(-1)
    out = np.empty(p.size * 2, dtype=np.uint8)
    out[0::2] = p & 0xF
    out[1::2] = p >> 4
    return out[:n]


@dataclasses.dataclass
class OracleQuant:
    fmt: str
    rows: int
    cols: int
    group: int
    hadamard: int | None
    element_codes: np.ndarray   # uint8 [rows, cols]
    scale_codes: np.ndarray     # uint8 [rows, cols // group]
    tensor_scale: float         # float32-valued
    mse_rel: float
    mse_top_rel: float

    @property
    def codes(self) -> np.ndarray:
        """Packed codes, uint8 [rows, cols // 2] (row-major = MfpTensor.codes)."""
        return pack_nibbles(self.element_codes).reshape(self.rows, -1)

    def group_scales(self) -> np.ndarray:
        if self.fmt == MXFP4:
            return np.ldexp(1.0, self.scale_codes.astype(np.int64) - 127)
        return E4M3_LEVELS[self.scale_codes.astype(np.intp)]


def _format_params(fmt: str):
    if fmt == MXFP4:
        return 32
    if fmt == NVFP4:
        return 16
    raise OracleDataError(f"unknown format {fmt!r}")


def quantize_rtn(X, fmt: str, hadamard: int | None = None,
                 four_thirds: bool = True, static_ts: float | None = None) -> OracleQuant:
    """RTN quantization with absmax scales, optionally Hadamard-rotated.

    Restates ``quantize_rtn`` (quantizers.py:247-255) for the two hardware
    formats: MXFP4 = (G=32, E8M0, tensor scale f32(4/3)) and NVFP4 = (G=16,
    E4M3, whole-tensor global scale), FormatSpec presets formats.py:301-307.
    """
    G = _format_params(fmt)
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] < 1 or X.shape[1] < 1:           # quantizers.py:97-98
        raise OracleDataError("expected a non-empty 2-D matrix")
    if not np.isfinite(X).all():                                   # quantizers.py:99-100
        raise OracleDataError("non-finite element")
    rows, cols = X.shape
    if cols % G:                                                   # quantizers.py:106-107
        raise OracleDataError(f"columns ({cols}) not divisible by group size ({G})")
    if hadamard and cols % hadamard:                               # quantizers.py:108-111
        raise OracleDataError(f"columns ({cols}) not divisible by transform block ({hadamard})")
    Y = rotate_blockwise(X, hadamard)
    B = Y.reshape(rows, cols // G, G)
    amax = np.abs(B).max(axis=2)                                   # quantizers.py:177
    raw = np.where(amax == 0.0, 1.0, amax / 6.0)                   # quantizers.py:187
    if fmt == NVFP4:                                               # quantizers.py:198-200
        top = float(amax.max()) / 6.0
        s_glob = float(np.float32(top / E4M3_MAX)) if top > 0 else 1.0
        if static_ts is not None:   # a given s_global: _encode_raw / _quantize_groups (:157-167, :211-215)
            s_glob = float(np.float32(static_ts))
        scodes = e4m3_encode(raw / s_glob)                         # quantizers.py:162-167
        dec = E4M3_LEVELS[scodes.astype(np.intp)]
        ts = float(np.float32(s_glob))                             # quantizers.py:191
    else:
        scodes = e8m0_encode(raw)
        dec = np.ldexp(1.0, scodes.astype(np.int64) - 127)
        ts = FOUR_THIRDS_F32 if four_thirds else 1.0               # quantizers.py:203-207
    eff = ts * dec                                                 # quantizers.py:90-92
    with np.errstate(divide="ignore", invalid="ignore"):
        u = B / eff[..., None]                                     # quantizers.py:213
    ecodes = fp4_codes(u)
    vals = eff[..., None] * fp4_values(ecodes)
    mse_rel, mse_top = _metrics(B, vals)
    return OracleQuant(fmt, rows, cols, G, hadamard or None,
                       ecodes.reshape(rows, cols), scodes, ts, mse_rel, mse_top)


def _metrics(B, Bh) -> tuple[float, float]:
    """mse_rel and mse_top_rel in the rotated domain (quantizers.py:218-231)."""
    den = float((B ** 2).sum())
    mse = float(((B - Bh) ** 2).sum() / den) if den > 0 else 0.0
    b2 = B.reshape(-1, B.shape[-1])
    h2 = Bh.reshape(-1, B.shape[-1])
    arg = np.argmax(np.abs(b2), axis=1)
    r = np.arange(b2.shape[0])
    top = b2[r, arg]
    t2 = top ** 2
    e2 = (top - h2[r, arg]) ** 2
    ratio = np.divide(e2, t2, out=np.zeros_like(e2), where=t2 > 0)
    return mse, float(ratio.mean())


def dequantize(q: OracleQuant) -> np.ndarray:
    """ts * scale * fp4 in float64  (formats.py:424-442)."""
    vals = fp4_values(q.element_codes).reshape(q.rows, q.cols // q.group, q.group)
    out = q.tensor_scale * q.group_scales()[:, :, None] * vals
    return out.reshape(q.rows, q.cols)


def linear_reference(Aq: OracleQuant, Wq: OracleQuant) -> np.ndarray:
    """Y = dequantize(Aq).astype(f32) @ dequantize(Wq).astype(f32).T."""
    a = dequantize(Aq).astype(np.float32)
    w = dequantize(Wq).astype(np.float32)
    return a @ w.T


# --- tensor-core scale-factor layout (hardware fact) ---

def sf_swizzled_size(rows: int, sf_cols: int) -> int:
    return (-(-rows // 128) * 128) * (-(-sf_cols // 4) * 4)


def _sf_offsets(rows: int, sf_cols: int) -> np.ndarray:
    r = np.arange(rows)[:, None]
    c = np.arange(sf_cols)[None, :]
    cb = -(-sf_cols // 4)
    return ((r // 128) * cb + c // 4) * 512 + (r % 32) * 16 + ((r // 32) % 4) * 4 + (c % 4)


def sf_swizzle(sf) -> np.ndarray:
    """Row-major [rows, sf_cols] scale codes -> padded 128x4-atom blocked bytes."""
    sf = np.asarray(sf, dtype=np.uint8)
    rows, cols = sf.shape
    out = np.zeros(sf_swizzled_size(rows, cols), dtype=np.uint8)
    out[_sf_offsets(rows, cols)] = sf
    return out


def sf_unswizzle(buf, rows: int, sf_cols: int) -> np.ndarray:
    return np.asarray(buf, dtype=np.uint8)[_sf_offsets(rows, sf_cols)]


# --- MFPQ container bytes (fileio.py:138-167), for the golden-hash pin ------

def mfpq_bytes(q: OracleQuant) -> bytes:
    scale_tag = "e8m0" if q.fmt == MXFP4 else "e4m3"
    tr = f"hadamard:{q.hadamard}" if q.hadamard else "none"
    header = "".join(f"{k}={v}\n" for k, v in [
        ("group_size", q.group), ("element", "fp4_e2m1"), ("scale", scale_tag),
        ("global_scale", int(q.fmt == NVFP4)), ("rows", q.rows), ("cols", q.cols),
        ("tensor_scale", float(q.tensor_scale).hex()), ("transform", tr), ("perm", 0),
    ]).encode()
    return b"".join([b"MFPQ", struct.pack("<BI", 1, len(header)), header,
                     pack_nibbles(q.element_codes).tobytes(),
                     np.asarray(q.scale_codes, dtype=np.uint8).reshape(-1).tobytes()])


def bf16_round(x) -> np.ndarray:
    """Round to the nearest bf16 (ties to even); returns float32 values."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).reshape(f.shape)


# --- multi-threaded variant used for the CPU baseline (same results, no metrics) ---

def quantize_rtn_parallel(X, fmt: str, hadamard: int | None = None, workers: int | None = None,
                          rows_per_chunk: int = 64) -> OracleQuant:
    """``quantize_rtn`` split over row chunks on a thread pool (numpy releases the GIL).

    Identical codes / scales / tensor scale to :func:`quantize_rtn`; the NVFP4
    whole-tensor max (quantizers.py:198-200) is a reduction over the chunk maxima.
    Metrics are not computed (mse_rel = mse_top_rel = nan).
    """
    import concurrent.futures as cf
    import os

    G = _format_params(fmt)
    X = np.asarray(X)
    rows, cols = X.shape
    if cols % G or (hadamard and cols % hadamard):
        raise OracleDataError("columns not divisible by group size / transform block")
    workers = workers or os.cpu_count() or 1
    bounds = [(r, min(r + rows_per_chunk, rows)) for r in range(0, rows, rows_per_chunk)]
    ecodes = np.empty((rows, cols), np.uint8)
    scodes = np.empty((rows, cols // G), np.uint8)
    amax = np.empty((rows, cols // G))

    def phase1(b):
        Xc = np.asarray(X[b[0]:b[1]], dtype=np.float64)
        if not np.isfinite(Xc).all():
            raise OracleDataError("non-finite element")
        Y = rotate_blockwise(Xc, hadamard)
        amax[b[0]:b[1]] = np.abs(Y.reshape(len(Y), -1, G)).max(axis=2)
        return Y

    with cf.ThreadPoolExecutor(workers) as ex:
        Ys = list(ex.map(phase1, bounds))
        if fmt == NVFP4:
            top = float(amax.max()) / 6.0
            s_glob = float(np.float32(top / E4M3_MAX)) if top > 0 else 1.0
            ts = s_glob
        else:
            s_glob, ts = 1.0, FOUR_THIRDS_F32

        def phase2(i):
            r0, r1 = bounds[i]
            am = amax[r0:r1]
            raw = np.where(am == 0.0, 1.0, am / 6.0)
            if fmt == NVFP4:
                sc = e4m3_encode(raw / s_glob)
                dec = E4M3_LEVELS[sc.astype(np.intp)]
            else:
                sc = e8m0_encode(raw)
                dec = np.ldexp(1.0, sc.astype(np.int64) - 127)
            eff = ts * dec
            with np.errstate(divide="ignore", invalid="ignore"):
                u = Ys[i].reshape(r1 - r0, -1, G) / eff[..., None]
            ecodes[r0:r1] = fp4_codes(u).reshape(r1 - r0, cols)
            scodes[r0:r1] = sc

        list(ex.map(phase2, range(len(bounds))))
    return OracleQuant(fmt, rows, cols, G, hadamard or None, ecodes, scodes, ts, float("nan"), float("nan"))


def dequantize_f32(q: OracleQuant) -> np.ndarray:
    """dequantize(q).astype(float32) (formats.py:441 in float64, then cast)."""
    return dequantize(q).astype(np.float32)
