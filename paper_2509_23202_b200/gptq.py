"""GPU GPTQ / MR-GPTQ: drop-in for microfp.gptq's solver
(/root/reference/pkg/src/microfp/gptq.py), same names, argument meaning and exceptions.

Pipeline, as ``gptq_quantize`` (gptq.py:181-238) runs it, all on the device in float64:
  fuse the transform into W (``mrfp4_rotate_f64``, transforms.py:77-91) and conjugate H
  (blockwise U^T H U, gptq.py:170-178) -> group scales on the current column order (absmax:
  the float64 ``quantize_rtn`` path; MSE: ``mse_optimize_scales``; fitted E8M0 grid:
  quantizers.py:128-154) -> static act-order permutation (gptq.py:113-116) -> dampening
  (:119-129) -> upper inverse-Cholesky factor T (:125-134, cuSOLVER) -> column-serial
  quantization with lazy block updates (:148-167): each block of <= 128 columns is solved by
  ``mrfp4_gptq_block`` (one thread per row, the reference's unfused float64 operations), the
  trailing update W[:, i2:] -= Err @ T[i1:i2, i2:] is a float64 GEMM -> un-permute, pack.

Parity: the float64 linear algebra (Cholesky, GEMM summation order) differs from
numpy/OpenBLAS/LAPACK in the last bits, and GPTQ's rounding decisions propagate them, so the
bar is the reference's objective: the proxy loss (gptq.py:303-311) of the result
(tests/test_gpu_gptq.py, fixtures from the reference solver).
"""

from __future__ import annotations

import dataclasses

import numpy as np
import torch

from . import _lib
from .errors import DataError, NumericalError
from .formats import FMT_NVFP4, GROUP, MfpTensor, ScaleMode, ScalePolicy, format_code
from .quantize import (GpuQuantResult, _quantize_rtn_f64, alloc_result, as_device_matrix, mse_optimize_scales,
                       rotate_f64)
from .transforms import TransformSpec, hadamard_block

__all__ = ["GptqConfig", "Hessian", "accumulate_hessian", "gptq_quantize", "mr_gptq", "proxy_loss",
           "static_act_order", "dampened_hessian", "conjugated_hessian", "GpuGptqResult"]

_E4M3_LEVELS = None


@dataclasses.dataclass
class GptqConfig:
    """gptq.py:51-63 (same fields and validation)."""

    dampening: float = 1e-2
    block_width: int = 128
    act_order: bool = False
    scale_policy: ScalePolicy = dataclasses.field(default_factory=ScalePolicy)
    transform: TransformSpec | None = None

    def __post_init__(self):
        if self.dampening <= 0:
            raise DataError("dampening must be positive")
        if self.block_width < 1:
            raise DataError("block width must be positive")


class Hessian:
    """Device accumulator for 2 X^T X over calibration batches (gptq.py:66-79)."""

    def __init__(self, n_cols: int, device="cuda"):
        self.matrix = torch.zeros((n_cols, n_cols), dtype=torch.float64, device=device)
        self.sample_count = 0

    @property
    def n_cols(self) -> int:
        return self.matrix.shape[0]

    def finalized(self) -> torch.Tensor:
        return self.matrix / max(self.sample_count, 1)


def accumulate_hessian(X_batch, state: Hessian) -> Hessian:
    """gptq.py:82-95 on the device: H += 2 X^T X (float64 GEMM)."""
    X = torch.as_tensor(np.asarray(X_batch, dtype=np.float64) if not isinstance(X_batch, torch.Tensor) else X_batch)
    X = X.to(device=state.matrix.device, dtype=torch.float64)
    if X.dim() != 2 or X.shape[1] != state.n_cols:
        raise DataError(f"batch with {X.shape[-1] if X.dim() == 2 else '?'} columns "
                        f"does not match Hessian size {state.n_cols}")
    if not bool(torch.isfinite(X).all()):
        raise DataError("non-finite element in calibration batch")
    state.matrix += 2.0 * (X.T @ X)
    state.sample_count += X.shape[0]
    return state


def _hessian_matrix(H, device) -> torch.Tensor:
    """Hessian object (this module's or the reference's), ndarray or tensor -> device float64 (gptq.py:98-105)."""
    if hasattr(H, "finalized"):
        H = H.finalized()
    Hm = torch.as_tensor(H if isinstance(H, torch.Tensor) else np.asarray(H, dtype=np.float64))
    Hm = Hm.to(device=device, dtype=torch.float64)
    if Hm.dim() != 2 or Hm.shape[0] != Hm.shape[1]:
        raise DataError("Hessian must be square")
    return Hm


def static_act_order(Hm: torch.Tensor) -> torch.Tensor:
    """Column permutation by descending Hessian diagonal, stable ties (gptq.py:108-111)."""
    return torch.argsort(-torch.diagonal(Hm), stable=True)


def dampened_hessian(Hm: torch.Tensor, cfg: GptqConfig) -> torch.Tensor:
    """Dead diagonals -> mean, then + dampening * mean * I (gptq.py:114-122)."""
    Hd = Hm.clone()
    d = torch.diagonal(Hd).clone()
    mean0 = float(d.mean())
    if mean0 <= 0:
        mean0 = 1.0
    d[d == 0] = mean0
    torch.diagonal(Hd).copy_(d + cfg.dampening * float(d.mean()))
    return Hd


def _inverse_factor(Hd: torch.Tensor) -> torch.Tensor:
    """Upper-triangular T with inv(Hd) = T^T T (gptq.py:125-134)."""
    L, info = torch.linalg.cholesky_ex(Hd)
    if int(info) != 0:
        raise NumericalError("Hessian Cholesky failed even after dampening; increase the dampening factor")
    Hinv = torch.cholesky_inverse(L)
    T, info = torch.linalg.cholesky_ex(Hinv, upper=True)
    if int(info) != 0:
        raise NumericalError("Hessian Cholesky failed even after dampening; increase the dampening factor")
    return T.contiguous()


def _sylvester_unit(k: int, device) -> torch.Tensor:
    idx = torch.arange(k, device=device)
    a = idx[:, None] & idx[None, :]
    par = torch.zeros((k, k), dtype=torch.int64, device=device)
    while bool(a.any()):
        par ^= a & 1
        a = a >> 1
    return (1 - 2 * par).to(torch.float64) / float(np.sqrt(k))   # _sylvester(k) / np.sqrt(k)


def conjugated_hessian(Hm: torch.Tensor, transform: TransformSpec | None) -> torch.Tensor:
    """Ubd^T H Ubd for the block-diagonal Ubd = I (x) U (gptq.py:170-178), blockwise."""
    k = hadamard_block(transform)
    if not k:
        return Hm
    d = Hm.shape[0]
    if d % k:
        raise DataError(f"Hessian size ({d}) not divisible by transform block ({k})")
    U = _sylvester_unit(k, Hm.device)
    nb = d // k
    H4 = Hm.reshape(nb, k, nb, k)
    return torch.einsum("ai,xayb,bj->xiyj", U, H4, U).reshape(d, d).contiguous()


def _decode(codes: torch.Tensor, fmt: int) -> torch.Tensor:
    global _E4M3_LEVELS
    if fmt == FMT_NVFP4:
        if _E4M3_LEVELS is None or _E4M3_LEVELS.device != codes.device:
            c = torch.arange(128, dtype=torch.float64)
            e, m = torch.div(c, 8, rounding_mode="floor"), torch.remainder(c, 8)
            lv = torch.where(e == 0, m * 2.0 ** -9, (1.0 + m / 8.0) * torch.pow(2.0, e - 7))
            _E4M3_LEVELS = lv.to(codes.device)
        return _E4M3_LEVELS[codes.long()]
    return torch.pow(2.0, codes.to(torch.float64) - 127.0)


@dataclasses.dataclass
class _Scales:
    codes: torch.Tensor      # uint8 [rows, cols / G]
    decoded: torch.Tensor    # float64 [rows, cols / G]
    tensor_scale: float
    fit: tuple | None


def _group_scales(Wt: torch.Tensor, fmt: int, policy: ScalePolicy) -> _Scales:
    """prepare_scales / optimize_group_scales of the rotated weight (quantizers.py:170-208, :263-327)."""
    spec_fmt = fmt
    rows, cols = Wt.shape
    G = GROUP[fmt]
    fit = getattr(policy, "scale_fit", None)
    if fit is not None:
        if fmt == FMT_NVFP4:
            raise DataError("scale_fit is only valid with the E8M0 scale format")
        absmax = Wt.view(rows, cols // G, G).abs().amax(dim=2)
        raw = torch.where(absmax == 0, torch.ones_like(absmax), absmax / 6.0)
        if fit == "auto":                                              # fit_e8m0_range, quantizers.py:128-141
            lo, hi = float(torch.log2(raw.min())), float(torch.log2(raw.max()))
            fit = ((hi - lo) / 255.0, lo)
        alpha, beta = (float(fit[0]), float(fit[1]))
        if alpha == 0.0:                                               # _fit_encode / _fit_decode (:144-154)
            codes = torch.zeros_like(raw, dtype=torch.uint8)
        else:
            codes = torch.clamp(torch.round((torch.log2(raw) - beta) / alpha), 0, 255).to(torch.uint8)
        dec = torch.exp2(alpha * codes.to(torch.float64) + beta)
        return _Scales(codes, dec, 1.0, (alpha, beta))
    if getattr(getattr(policy, "mode", None), "value", "absmax") == "mse":
        r = mse_optimize_scales(Wt, _spec(spec_fmt), policy=policy)
    else:
        r = _quantize_rtn_f64(Wt, fmt, 0, bool(getattr(policy, "e8m0_four_thirds", True)), None, True)
    sc = r.scale_codes()
    return _Scales(sc, _decode(sc, fmt), r.tensor_scale, None)


def _spec(fmt: int):
    from .formats import spec_for
    return spec_for(fmt)


class GpuGptqResult(GpuQuantResult):
    """GpuQuantResult of the solver, plus the act-order permutation (MFPQ section) and the
    fitted E8M0 grid when the policy asked for one (not GEMM-consumable)."""

    perm: torch.Tensor | None = None
    scale_fit: tuple | None = None

    def to_mfp(self) -> MfpTensor:
        if self.scale_fit is None:
            return super().to_mfp()
        sc = self.scale_codes_raw.reshape(-1).cpu().numpy()
        return MfpTensor(self.spec, self.rows, self.cols, self.codes.reshape(-1).cpu().numpy(), sc,
                         self.tensor_scale, self.transform, self.scale_fit)


def _core(Wp: torch.Tensor, T: torch.Tensor, Sp: torch.Tensor, block_width: int):
    """_gptq_core (gptq.py:148-167) on the device; returns (Q, codes) in the permuted order."""
    rows, d = Wp.shape
    W = Wp.clone().contiguous()
    Sp = Sp.contiguous()
    Q = torch.empty_like(W)
    codes = torch.empty((rows, d), dtype=torch.uint8, device=W.device)
    Err = torch.empty((rows, 128), dtype=torch.float64, device=W.device)
    L = _lib.lib()
    stream = _lib.stream_ptr(torch, W.device)
    bw = min(block_width, 128)
    for i1 in range(0, d, bw):
        i2 = min(i1 + bw, d)
        _lib.check(L.mrfp4_gptq_block(_lib.ptr(W), _lib.ptr(Sp), _lib.ptr(T), rows, d, i1, i2 - i1, _lib.ptr(Q),
                                      _lib.ptr(codes), _lib.ptr(Err), stream))
        if i2 < d:
            W[:, i2:].sub_(Err[:, :i2 - i1] @ T[i1:i2, i2:])
    return Q, codes


def _metrics(Xt: torch.Tensor, Xh: torch.Tensor, G: int):
    """_matrix_metrics (quantizers.py:218-231), float64."""
    err2 = float(((Xt - Xh) ** 2).sum())
    denom = float((Xt ** 2).sum())
    B, Bh = Xt.reshape(-1, G), Xh.reshape(-1, G)
    it = B.abs().argmax(dim=1, keepdim=True)
    top, qt = B.gather(1, it).squeeze(1), Bh.gather(1, it).squeeze(1)
    t2 = top * top
    ratio = torch.where(t2 > 0, (top - qt) ** 2 / torch.where(t2 > 0, t2, torch.ones_like(t2)), torch.zeros_like(t2))
    return (err2 / denom if denom > 0 else 0.0), float(ratio.mean())


def gptq_quantize(W, H, spec, cfg: GptqConfig | None = None, *, device="cuda") -> GpuGptqResult:
    """GPTQ of a weight against a calibration Hessian, on the GPU (gptq.py:181-238).
    Returns a GpuGptqResult: device codes / swizzled scales / tensor scale (``prepare_weight``
    consumes it unless a fitted E8M0 grid was requested), ``.to_mfp()``, ``.mse_rel``,
    ``.mse_top_rel`` and the act-order ``.perm``."""
    cfg = cfg or GptqConfig()
    fmt = format_code(spec)
    if not isinstance(W, torch.Tensor):
        W = torch.from_numpy(np.ascontiguousarray(np.asarray(W, dtype=np.float64)))
    if W.dim() != 2:
        raise DataError("expected a 2-D weight matrix")
    W = W.to(device=device, dtype=torch.float64).contiguous()
    if not bool(torch.isfinite(W).all()):
        raise DataError("non-finite element in weights")
    rows, cols = W.shape
    G = GROUP[fmt]
    if cols % G:
        raise DataError(f"columns ({cols}) not divisible by group size ({G})")
    Hm = _hessian_matrix(H, W.device)
    if Hm.shape[0] != cols:
        raise DataError("Hessian size does not match the weight columns")
    had_k = hadamard_block(cfg.transform)
    if had_k:
        if cols % had_k:
            raise DataError(f"columns ({cols}) not divisible by transform block ({had_k})")
        Wt = rotate_f64(W, had_k)
        Hm = conjugated_hessian(Hm, cfg.transform)
    else:
        Wt = W
    sc = _group_scales(Wt, fmt, cfg.scale_policy)
    col_scales = (sc.tensor_scale * sc.decoded).repeat_interleave(G, dim=1)[:, :cols]   # gptq.py:137-140
    if cfg.act_order:
        perm = static_act_order(Hm)
        Wp, Hp, Sp = Wt[:, perm], Hm[perm][:, perm], col_scales[:, perm]
    else:
        perm = None
        Wp, Hp, Sp = Wt, Hm, col_scales
    T = _inverse_factor(dampened_hessian(Hp, cfg))
    Q, codes = _core(Wp, T, Sp, cfg.block_width)
    if perm is not None:
        inv = torch.argsort(perm)
        Q, codes = Q[:, inv], codes[:, inv]
    packed = (codes[:, 0::2] | (codes[:, 1::2] << 4)).contiguous()
    base = alloc_result(rows, cols, fmt, had_k, W.device)
    res = GpuGptqResult(fmt, rows, cols, had_k, packed, base.sf, base.tensor_scale_dev, base.scratch)
    L = _lib.lib()
    with torch.cuda.device(W.device):
        _lib.check(L.mrfp4_sf_swizzle(_lib.ptr(sc.codes.contiguous()), _lib.ptr(res.sf), rows, cols // G,
                                      _lib.stream_ptr(torch, W.device)))
    res.tensor_scale_dev.fill_(float(np.float32(sc.tensor_scale)))
    res.perm = perm
    res.scale_fit = sc.fit
    res.scale_codes_raw = sc.codes
    res._metrics = _metrics(Wt, Q, G)
    return res


def mr_gptq(W, H, spec, cfg: GptqConfig | None = None, transform: TransformSpec | None = None,
            *, device="cuda") -> GpuGptqResult:
    """Micro-rotated GPTQ (gptq.py:274-300): Hadamard block = group size by default, MSE scales
    for E4M3 formats, absmax + fitted E8M0 grid for MXFP4 (not hardware E8M0: pass
    ``cfg.scale_policy`` via gptq_quantize for the hardware MR-MXFP4), static act-order."""
    base = cfg or GptqConfig()
    if transform is None:
        transform = base.transform
    if transform is None:
        transform = TransformSpec.hadamard(GROUP[format_code(spec)])
    fmt = format_code(spec)
    if fmt != FMT_NVFP4 and hadamard_block(transform) > 128:
        raise DataError("MR-GPTQ Hadamard blocks are limited to 128 for E8M0 formats")
    if fmt == FMT_NVFP4:
        policy = ScalePolicy(mode=ScaleMode.MSE)
    else:
        policy = ScalePolicy(mode=ScaleMode.ABSMAX, scale_fit="auto")
    forced = dataclasses.replace(base, transform=transform, scale_policy=policy, act_order=True)
    return gptq_quantize(W, H, spec, forced, device=device)


def proxy_loss(W, W_hat, H) -> float:
    """0.5 * sum((E @ H) * E) with the unnormalized Hessian (gptq.py:303-311), float64 on the device."""
    dev = W_hat.device if isinstance(W_hat, torch.Tensor) else "cuda"
    t = lambda a: (a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a, dtype=np.float64))).to(
        device=dev, dtype=torch.float64)
    M = H.matrix if hasattr(H, "matrix") else H
    E = t(W_hat) - t(W)
    return float(0.5 * ((E @ t(M)) * E).sum())
