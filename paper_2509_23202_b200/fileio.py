"""MFPQ quantized-container files -> the GPU weight path.

Byte layout of the reference's QuantFile (/root/reference/pkg/src/microfp/fileio.py:7-12,
writer :138-167, reader :170-226): b"MFPQ", u8 version (1), u32-LE header length,
UTF-8 ``key=value`` lines, then packed codes, one scale byte per group (float64
for unquantized scales) and an optional u64-LE column permutation.  The
permutation is informational: codes are stored in the original column order
(gptq.py:227-230, pkg/README.md:123-124), so the GPU path ignores it.

This lets ``microfp quantize ... --method mr-gptq --scale-opt absmax`` artefacts
feed ``prepare_weight`` with no Python re-quantization.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import DataError
from .formats import FormatSpec, MfpTensor, ScaleFormat, ScaleKind
from .transforms import TransformKind, TransformSpec

MAGIC = b"MFPQ"
VERSION = 1


def _scale_format(tag: str) -> ScaleFormat:
    if tag == "e8m0":
        return ScaleFormat.e8m0()
    if tag == "e4m3":
        return ScaleFormat.e4m3()
    if tag == "unquantized":
        return ScaleFormat.unquantized()
    if tag.startswith("fpem:"):
        e, m, b = (int(t) for t in tag[5:].split(","))
        return ScaleFormat.fpem(e, m, b)
    if tag.startswith("int8:"):
        lo, hi = (float.fromhex(t) for t in tag[5:].split(","))
        return ScaleFormat.int8_linear(lo, hi)
    raise DataError(f"unknown scale format tag {tag!r}")


def _scale_tag(fmt: ScaleFormat) -> str:
    if fmt.kind is ScaleKind.E8M0:
        return "e8m0"
    if fmt.kind is ScaleKind.FPEM:
        return "e4m3" if (fmt.exp_bits, fmt.mant_bits, fmt.bias) == (4, 3, 7) else \
            f"fpem:{fmt.exp_bits},{fmt.mant_bits},{fmt.bias}"
    if fmt.kind is ScaleKind.INT8_LINEAR:
        return f"int8:{float(fmt.lo).hex()},{float(fmt.hi).hex()}"
    return "unquantized"


def _transform(tag: str):
    if tag == "none":
        return None
    kind, _, block = tag.partition(":")
    try:
        return TransformSpec(TransformKind(kind), int(block))
    except ValueError as exc:
        raise DataError(f"unknown transform tag {tag!r}") from exc


def parse_quant(blob: bytes, name: str = "<bytes>"):
    """Parse MFPQ bytes -> (MfpTensor, permutation or None)."""
    if len(blob) < 9 or blob[:4] != MAGIC:
        raise DataError(f"{name}: not a QuantFile")
    version, hlen = struct.unpack_from("<BI", blob, 4)
    if version != VERSION:
        raise DataError(f"{name}: unsupported QuantFile version {version}")
    if len(blob) < 9 + hlen:
        raise DataError(f"{name}: truncated header")
    fields = dict(line.partition("=")[::2] for line in blob[9:9 + hlen].decode("utf-8").splitlines() if line)
    try:
        spec = FormatSpec(int(fields["group_size"]), _scale_format(fields["scale"]),
                          bool(int(fields["global_scale"])), fields.get("element", "fp4_e2m1"))
        rows, cols = int(fields["rows"]), int(fields["cols"])
        ts = float.fromhex(fields["tensor_scale"])
        transform = _transform(fields.get("transform", "none"))
        fit = None
        if "scale_fit" in fields:
            a, b = fields["scale_fit"].split(",")
            fit = (float.fromhex(a), float.fromhex(b))
        has_perm = bool(int(fields.get("perm", "0")))
    except (KeyError, ValueError) as exc:
        raise DataError(f"{name}: malformed header ({exc})") from exc
    pos = 9 + hlen
    n_codes = (rows * cols + 1) // 2
    n_groups = rows * (cols // spec.group_size)
    unq = spec.scale.kind is ScaleKind.UNQUANTIZED
    need = n_codes + n_groups * (8 if unq else 1) + (8 * cols if has_perm else 0)
    if len(blob) != pos + need:
        raise DataError(f"{name}: section size mismatch")
    codes = np.frombuffer(blob, np.uint8, n_codes, pos).copy()
    pos += n_codes
    if unq:
        scales = np.frombuffer(blob, "<f8", n_groups, pos).astype(np.float64)
        pos += 8 * n_groups
    else:
        scales = np.frombuffer(blob, np.uint8, n_groups, pos).copy()
        pos += n_groups
    perm = np.frombuffer(blob, "<u8", cols, pos).astype(np.int64) if has_perm else None
    return MfpTensor(spec, rows, cols, codes, scales, ts, transform, fit), perm


def read_quant(path):
    with open(path, "rb") as fh:
        return parse_quant(fh.read(), str(path))


def quant_bytes(t, perm=None) -> bytes:
    """Serialize an MfpTensor-like container in the MFPQ layout."""
    tr = t.transform
    tr_tag = "none" if tr is None or tr.kind.value == "identity" else f"{tr.kind.value}:{tr.block}"
    lines = [f"group_size={t.spec.group_size}", f"element={t.spec.element}",
             f"scale={_scale_tag(t.spec.scale)}", f"global_scale={int(t.spec.global_scale)}",
             f"rows={t.rows}", f"cols={t.cols}", f"tensor_scale={float(t.tensor_scale).hex()}",
             f"transform={tr_tag}"]
    if t.scale_fit is not None:
        lines.append(f"scale_fit={float(t.scale_fit[0]).hex()},{float(t.scale_fit[1]).hex()}")
    lines.append(f"perm={int(perm is not None)}")
    header = ("\n".join(lines) + "\n").encode()
    unq = t.spec.scale.kind is ScaleKind.UNQUANTIZED
    parts = [MAGIC, struct.pack("<BI", VERSION, len(header)), header,
             np.ascontiguousarray(t.codes, dtype=np.uint8).tobytes(),
             np.asarray(t.scale_codes, dtype="<f8" if unq else np.uint8).tobytes()]
    if perm is not None:
        parts.append(np.asarray(perm).astype("<u8").tobytes())
    return b"".join(parts)


def write_quant(path, t, perm=None) -> None:
    with open(path, "wb") as fh:
        fh.write(quant_bytes(t, perm))
