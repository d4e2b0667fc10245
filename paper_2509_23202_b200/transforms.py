"""Block-rotation descriptors, mirroring microfp.transforms.TransformSpec.

Reference: /root/reference/pkg/src/microfp/transforms.py:29-53 (kinds, the
power-of-two check for Hadamard blocks).  Only the descriptor lives on the host;
the rotation itself runs inside the K1 CUDA kernel (an in-register fast
Walsh-Hadamard transform, Sylvester order, scaled by 1/sqrt(k)).
"""

from __future__ import annotations

import dataclasses
import enum

from .errors import DataError

GPU_HADAMARD_BLOCKS = (16, 32, 64, 128)


class TransformKind(enum.Enum):
    IDENTITY = "identity"
    HADAMARD = "hadamard"
    DCT2 = "dct"
    DST2 = "dst"


@dataclasses.dataclass(frozen=True)
class TransformSpec:
    kind: TransformKind
    block: int

    def __post_init__(self):
        if self.block < 1:
            raise DataError("transform block size must be positive")
        if self.kind is TransformKind.HADAMARD and (self.block & (self.block - 1)):
            raise DataError(f"Hadamard block size must be a power of two, got {self.block}")

    @classmethod
    def identity(cls, block: int = 1) -> "TransformSpec":
        return cls(TransformKind.IDENTITY, block)

    @classmethod
    def hadamard(cls, block: int) -> "TransformSpec":
        return cls(TransformKind.HADAMARD, block)


def hadamard_block(transform) -> int:
    """Map a TransformSpec (ours or the reference's) to the kernel's had_k (0 = none).

    Accepts any object with ``kind`` (enum whose value is "identity"/"hadamard"/...)
    and ``block``, so reference ``microfp.transforms.TransformSpec`` instances work.
    """
    if transform is None:
        return 0
    kind = getattr(getattr(transform, "kind", None), "value", None)
    block = int(getattr(transform, "block", 0))
    if kind == "identity":
        return 0
    if kind == "hadamard":
        if block not in GPU_HADAMARD_BLOCKS:
            raise DataError(f"unsupported on GPU path: Hadamard block {block} "
                            f"(supported: {GPU_HADAMARD_BLOCKS})")
        return block
    raise DataError(f"unsupported on GPU path: transform {kind!r}")


def transform_for(had_k: int):
    return TransformSpec.hadamard(had_k) if had_k else None
