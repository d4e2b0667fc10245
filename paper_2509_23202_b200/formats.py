"""Format descriptors and the host-side quantized container, mirroring microfp.formats.

Reference definitions (paths under /root/reference/pkg/src/microfp):
  ScaleKind / ScaleFormat  formats.py:141-217
  FormatSpec (+ presets)   formats.py:286-307
  MfpTensor invariants     formats.py:310-374
  pack/unpack (low nibble first)  formats.py:377-421

Only MXFP4 (G=32, E8M0) and NVFP4 (G=16, E4M3 + global scale) have a tensor-core
format, so only those two specs map to a GPU format code; everything else is
representable here (for interchange) but rejected by the GPU entry points with
``DataError("unsupported on GPU path: ...")``.
"""

from __future__ import annotations

import dataclasses
import enum

import numpy as np

from .errors import DataError

FMT_MXFP4 = 0  # include/mrfp4.h MRFP4_FMT_MXFP4
FMT_NVFP4 = 1  # include/mrfp4.h MRFP4_FMT_NVFP4
GROUP = {FMT_MXFP4: 32, FMT_NVFP4: 16}


class ScaleKind(enum.Enum):
    E8M0 = "e8m0"
    FPEM = "fpem"
    INT8_LINEAR = "int8"
    UNQUANTIZED = "unquantized"


@dataclasses.dataclass(frozen=True)
class ScaleFormat:
    kind: ScaleKind
    exp_bits: int = 0
    mant_bits: int = 0
    bias: int = 0
    lo: float | None = None
    hi: float | None = None

    @classmethod
    def e8m0(cls) -> "ScaleFormat":
        return cls(ScaleKind.E8M0, 8, 0, 127)

    @classmethod
    def fpem(cls, exp_bits: int, mant_bits: int, bias: int | None = None) -> "ScaleFormat":
        if exp_bits < 1 or mant_bits < 0 or exp_bits + mant_bits > 7:
            raise DataError("FpEM requires e >= 1 and e + m <= 7 (sign bit unused)")
        return cls(ScaleKind.FPEM, exp_bits, mant_bits,
                   (1 << (exp_bits - 1)) - 1 if bias is None else bias)

    @classmethod
    def e4m3(cls) -> "ScaleFormat":
        return cls.fpem(4, 3)

    @classmethod
    def int8_linear(cls, lo: float | None = None, hi: float | None = None) -> "ScaleFormat":
        if lo is not None and hi is not None and hi < lo:
            raise DataError("Int8Linear calibration range must have hi >= lo")
        return cls(ScaleKind.INT8_LINEAR, lo=lo, hi=hi)

    @classmethod
    def unquantized(cls) -> "ScaleFormat":
        return cls(ScaleKind.UNQUANTIZED)

    @property
    def n_codes(self) -> int:
        return 1 << (self.exp_bits + self.mant_bits) if self.kind is ScaleKind.FPEM else 256


@dataclasses.dataclass(frozen=True)
class FormatSpec:
    group_size: int
    scale: ScaleFormat
    global_scale: bool = False
    element: str = "fp4_e2m1"

    def __post_init__(self):
        if self.group_size < 1:
            raise DataError("group size must be positive")
        if self.element != "fp4_e2m1":
            raise DataError("only the FP4 E2M1 element codec is supported")

    @classmethod
    def mxfp4(cls) -> "FormatSpec":
        return cls(32, ScaleFormat.e8m0(), False)

    @classmethod
    def nvfp4(cls) -> "FormatSpec":
        return cls(16, ScaleFormat.e4m3(), True)


def format_code(spec) -> int:
    """GPU format code of a FormatSpec (ours or the reference's, matched by value)."""
    scale = getattr(spec, "scale", None)
    kind = getattr(getattr(scale, "kind", None), "value", None)
    g = int(getattr(spec, "group_size", 0))
    glob = bool(getattr(spec, "global_scale", False))
    if getattr(spec, "element", "fp4_e2m1") != "fp4_e2m1":
        raise DataError("only the FP4 E2M1 element codec is supported")
    if kind == "e8m0" and g == 32 and not glob:
        return FMT_MXFP4
    if (kind == "fpem" and g == 16 and glob
            and (scale.exp_bits, scale.mant_bits, scale.bias) == (4, 3, 7)):
        return FMT_NVFP4
    raise DataError(f"unsupported on GPU path: format (G={g}, scale={kind}, global={glob}); "
                    "tensor cores take MXFP4 (G=32, E8M0) or NVFP4 (G=16, E4M3, global scale)")


def spec_for(fmt: int) -> FormatSpec:
    return FormatSpec.mxfp4() if fmt == FMT_MXFP4 else FormatSpec.nvfp4()


@dataclasses.dataclass(frozen=True)
class MfpTensor:
    """Host container with the reference's field names and invariants (formats.py:310-358)."""

    spec: FormatSpec
    rows: int
    cols: int
    codes: np.ndarray
    scale_codes: np.ndarray
    tensor_scale: float = 1.0
    transform: object | None = None
    scale_fit: tuple[float, float] | None = None

    def __post_init__(self):
        g = self.spec.group_size
        if self.rows < 1 or self.cols < 1 or self.cols % g:
            raise DataError(f"dims ({self.rows}, {self.cols}) not compatible with group size {g}")
        if self.scale_codes.size != self.rows * (self.cols // g):
            raise DataError(f"expected {self.rows * (self.cols // g)} scale codes, got {self.scale_codes.size}")
        if self.codes.size != (self.rows * self.cols + 1) // 2:
            raise DataError("packed code buffer has the wrong size")
        kind = self.spec.scale.kind
        if self.scale_fit is not None and kind is not ScaleKind.E8M0:
            raise DataError("scale_fit is only valid with the E8M0 scale format")
        if kind in (ScaleKind.E8M0, ScaleKind.FPEM) and self.scale_codes.size and self.scale_fit is None:
            top = 254 if kind is ScaleKind.E8M0 else self.spec.scale.n_codes - 2
            if int(np.max(self.scale_codes)) > top:
                raise DataError("reserved scale code in container")

    @property
    def n_groups(self) -> int:
        return self.rows * (self.cols // self.spec.group_size)

    def element_codes(self) -> np.ndarray:
        return unpack_codes(self.codes, self.rows * self.cols).reshape(self.rows, self.cols)


def pack_codes(codes) -> np.ndarray:
    flat = np.asarray(codes, dtype=np.uint8).reshape(-1)
    if flat.size & 1:
        flat = np.append(flat, np.uint8(0))
    return (flat[0::2] | (flat[1::2] << 4)).astype(np.uint8)


def unpack_codes(packed, n: int) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8).reshape(-1)
    out = np.stack([p & 0xF, p >> 4], axis=1).reshape(-1)
    return out[:n]


def pack_tensor(element_codes, scale_codes, spec: FormatSpec, dims=None, tensor_scale: float = 1.0,
                transform=None, scale_fit=None) -> MfpTensor:
    ec = np.asarray(element_codes)
    if dims is None:
        if ec.ndim != 2:
            raise DataError("dims required for non-2D element codes")
        dims = ec.shape
    rows, cols = int(dims[0]), int(dims[1])
    if ec.size != rows * cols:
        raise DataError("element code count does not match dims")
    if ec.size and (ec.min() < 0 or ec.max() > 15):
        raise DataError("element code out of range")
    sc = np.asarray(scale_codes).reshape(-1)
    if spec.scale.kind is not ScaleKind.UNQUANTIZED:
        sc = sc.astype(np.uint8)
    return MfpTensor(spec, rows, cols, pack_codes(ec), sc, float(np.float32(tensor_scale)),
                     transform, scale_fit)


def unpack_tensor(t) -> tuple[np.ndarray, np.ndarray]:
    return unpack_codes(t.codes, t.rows * t.cols).reshape(t.rows, t.cols), np.array(t.scale_codes, copy=True)


class ScaleMode(enum.Enum):
    """How group scales are chosen (quantizers.py:42-44)."""

    ABSMAX = "absmax"
    MSE = "mse"


@dataclasses.dataclass(frozen=True)
class ScalePolicy:
    """Scale policy with the reference's fields (quantizers.py:47-59).  ``scale_fit`` (fitted
    E8M0 grid) has no hardware encoding and is rejected by the GPU path."""

    mode: ScaleMode = ScaleMode.ABSMAX
    e8m0_four_thirds: bool = True
    scale_fit: tuple | str | None = None
