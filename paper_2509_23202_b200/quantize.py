"""GPU ``quantize_rtn`` -- drop-in for microfp.quantizers.quantize_rtn on the hot path.

Reference: /root/reference/pkg/src/microfp/quantizers.py:247-255 (and :341-347 for
``quantize``).  Same name, argument meaning and error behaviour (``DataError`` for
non-2-D / empty / non-finite input, indivisible shapes, unsupported policies),
computed by the K1 CUDA kernel behind ``mrfp4_act_quant``.  The result keeps the
device buffers in the layout the GEMM consumes (codes [M, K/2], swizzled scale
factors, device tensor scale) and converts to the reference container on demand
(``.tensor`` / ``.to_mfp()``).

Numerics: bf16 / fp16 / fp32 inputs are exact in the kernel's fp32 registers; a
float64 input is rounded to fp32 first (the reference works in float64).
"""

from __future__ import annotations

import dataclasses

import numpy as np
import torch

from . import _lib
from .errors import DataError
from .formats import FMT_NVFP4, GROUP, MfpTensor, format_code, spec_for
from .transforms import hadamard_block, transform_for

_DT = {torch.bfloat16: _lib.DT_BF16, torch.float16: _lib.DT_F16, torch.float32: _lib.DT_F32}


def _check_policy(policy, fmt: int) -> None:
    if policy is None:
        return
    mode = getattr(getattr(policy, "mode", None), "value", "absmax")
    if mode != "absmax":
        raise DataError("unsupported on GPU path: ScaleMode.MSE (offline weight-only search, "
                        "quantizers.py:263-327); quantize weights with the reference and use prepare_weight")
    if getattr(policy, "scale_fit", None) is not None:
        raise DataError("unsupported on GPU path: scale_fit (fitted E8M0 grid is not hardware E8M0)")
    if fmt != FMT_NVFP4 and not getattr(policy, "e8m0_four_thirds", True):
        raise DataError("unsupported on GPU path: e8m0_four_thirds=False")


def as_device_matrix(X, device=None) -> torch.Tensor:
    """Validate like quantizers.py:95-101 (2-D, non-empty) and move to the GPU."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_23202_b200 needs a CUDA device (sm_100a); there is no CPU path")
    if not isinstance(X, torch.Tensor):
        X = torch.from_numpy(np.ascontiguousarray(np.asarray(X)))
    if X.dim() != 2 or X.shape[0] < 1 or X.shape[1] < 1:
        raise DataError("expected a non-empty 2-D matrix")
    if X.dtype == torch.float64:
        X = X.to(torch.float32)
    elif X.dtype not in _DT:
        X = X.to(torch.float32)
    if X.device.type != "cuda":
        X = X.to(device or "cuda", non_blocking=False)
    es = X.element_size()
    if X.stride(1) != 1 or (X.stride(0) * es) % 16 or X.data_ptr() % 16:
        X = X.contiguous()
        if (X.stride(0) * es) % 16:  # odd row length: pad the row stride
            pad = torch.zeros((X.shape[0], -(-X.shape[1] * es // 16) * 16 // es), dtype=X.dtype, device=X.device)
            pad[:, : X.shape[1]] = X
            X = pad[:, : X.shape[1]]
    return X


@dataclasses.dataclass
class GpuQuantResult:
    """Device-resident QuantResult: codes + swizzled scales + tensor scale (+ status)."""

    fmt: int
    rows: int
    cols: int
    had_k: int
    codes: torch.Tensor            # uint8 [rows, cols // 2]
    sf: torch.Tensor               # uint8, swizzled 128x4-atom layout
    tensor_scale_dev: torch.Tensor  # float32 [1]
    scratch: torch.Tensor          # int32 [12]: [0] status bits, [4:12] act-quant workspace (32 B)
    source: torch.Tensor | None = None   # the input X (for the lazily computed metrics)
    _metrics: tuple | None = None

    @property
    def spec(self):
        return spec_for(self.fmt)

    @property
    def transform(self):
        return transform_for(self.had_k)

    @property
    def group_size(self) -> int:
        return GROUP[self.fmt]

    @property
    def status(self) -> int:
        return int(self.scratch[0].item())

    def check(self) -> "GpuQuantResult":
        s = self.status
        if s & (_lib.STATUS_NONFINITE | _lib.STATUS_SCALE_UNDERFLOW):
            raise DataError("non-finite element")  # quantizers.py:99-100 / formats.py:101-102
        return self

    @property
    def tensor_scale(self) -> float:
        return float(self.tensor_scale_dev.item())

    def scale_codes(self) -> torch.Tensor:
        """Row-major [rows, cols // G] scale codes on the device (unswizzled)."""
        out = torch.empty((self.rows, self.cols // self.group_size), dtype=torch.uint8, device=self.codes.device)
        _lib.check(_lib.lib().mrfp4_sf_unswizzle(_lib.ptr(self.sf), _lib.ptr(out), self.rows, out.shape[1],
                                                 _lib.stream_ptr(torch, self.codes.device)))
        return out

    def to_mfp(self) -> MfpTensor:
        """Reference-layout host container (MfpTensor: formats.py:310-358)."""
        return MfpTensor(self.spec, self.rows, self.cols, self.codes.reshape(-1).cpu().numpy(),
                         self.scale_codes().reshape(-1).cpu().numpy(), self.tensor_scale,
                         self.transform, None)

    @property
    def tensor(self) -> MfpTensor:
        return self.to_mfp()

    def metrics(self) -> tuple[float, float]:
        """(mse_rel, mse_top_rel) of the reference's QuantResult (quantizers.py:218-231),
        computed on the device in fp64 in the rotated domain (first call synchronizes)."""
        if self._metrics is None:
            if self.source is None:
                raise DataError("metrics need the quantized input (result built without a source)")
            X = self.source
            acc = torch.zeros(3, dtype=torch.float64, device=self.codes.device)
            _lib.check(_lib.lib().mrfp4_quant_metrics(
                _lib.ptr(X), _DT[X.dtype], self.rows, self.cols, X.stride(0), self.fmt, self.had_k,
                _lib.ptr(self.codes), _lib.ptr(self.sf), _lib.ptr(self.tensor_scale_dev), _lib.ptr(acc),
                _lib.stream_ptr(torch, X.device)))
            e2, x2, top = acc.tolist()
            n_groups = self.rows * (self.cols // self.group_size)
            self._metrics = (e2 / x2 if x2 > 0 else 0.0, top / n_groups)
        return self._metrics

    @property
    def mse_rel(self) -> float:
        return self.metrics()[0]

    @property
    def mse_top_rel(self) -> float:
        return self.metrics()[1]


def act_quant_into(X: torch.Tensor, fmt: int, had_k: int, codes: torch.Tensor, sf: torch.Tensor,
                   ts: torch.Tensor, scratch: torch.Tensor) -> None:
    """Launch K1 on the current stream into caller-provided buffers (no allocation)."""
    M, K = X.shape
    L = _lib.lib()
    _lib.check(L.mrfp4_act_quant(_lib.ptr(X), _DT[X.dtype], M, K, X.stride(0), fmt, had_k,
                                 _lib.ptr(codes), _lib.ptr(sf), _lib.ptr(ts), _lib.ptr(scratch),
                                 _lib.ptr(scratch) + 16, 32, _lib.stream_ptr(torch, X.device)))


def alloc_result(M: int, K: int, fmt: int, had_k: int, device) -> GpuQuantResult:
    G = GROUP[fmt]
    sfb = _lib.lib().mrfp4_sf_bytes(M, K // G)
    return GpuQuantResult(
        fmt, M, K, had_k,
        torch.empty((M, K // 2), dtype=torch.uint8, device=device),
        torch.empty(sfb, dtype=torch.uint8, device=device),
        torch.empty(1, dtype=torch.float32, device=device),
        torch.zeros(12, dtype=torch.int32, device=device))


def quantize_rtn(X, spec, policy=None, transform=None, *, check: bool = True) -> GpuQuantResult:
    """Round-to-nearest FP4 quantization with absmax scales, on the GPU.

    Drop-in for ``microfp.quantize_rtn`` (quantizers.py:247-255) for the MXFP4 /
    NVFP4 presets and Hadamard blocks 16/32/64/128 (or no transform).
    ``check=True`` (the reference behaviour) synchronizes to raise ``DataError`` on
    non-finite data; pass ``check=False`` to stay asynchronous and call
    ``.check()`` later.
    """
    fmt = format_code(spec)
    _check_policy(policy, fmt)
    had_k = hadamard_block(transform)
    X = as_device_matrix(X)
    M, K = X.shape
    G = GROUP[fmt]
    if K % G:                                                       # quantizers.py:106-107
        raise DataError(f"columns ({K}) not divisible by group size ({G})")
    if had_k and K % had_k:                                         # quantizers.py:108-111
        raise DataError(f"columns ({K}) not divisible by transform block ({had_k})")
    res = alloc_result(M, K, fmt, had_k, X.device)
    act_quant_into(X, fmt, had_k, res.codes, res.sf, res.tensor_scale_dev, res.scratch)
    res.source = X
    if check:
        res.check()
    return res


def quantize(X, spec, policy=None, transform=None, *, check: bool = True) -> GpuQuantResult:
    """``microfp.quantize`` dispatch (quantizers.py:341-347); MSE mode is offline-only."""
    return quantize_rtn(X, spec, policy=policy, transform=transform, check=check)
