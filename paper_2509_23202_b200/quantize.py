"""GPU ``quantize_rtn`` -- drop-in for microfp.quantizers.quantize_rtn on the hot path.

Reference: /root/reference/pkg/src/microfp/quantizers.py:247-255 (and :341-347 for
``quantize``).  Same name, argument meaning and error behaviour (``DataError`` for
non-2-D / empty / non-finite input, indivisible shapes, unsupported policies),
computed by the K1 CUDA kernel behind ``mrfp4_act_quant``.  The result keeps the
device buffers in the layout the GEMM consumes (codes [M, K/2], swizzled scale
factors, device tensor scale) and converts to the reference container on demand
(``.tensor`` / ``.to_mfp()``).

Numerics: bf16 / fp16 / fp32 inputs are exact in the kernel's fp32 registers.  A float64
input (the reference's own dtype, quantizers.py:96) takes a float64 device path instead:
``mrfp4_rotate_f64`` (the reference's summation order) and the float64 encoder of
``mrfp4_mse_pass`` with the single candidate 1.0 -- prepare_scales + _assemble
(quantizers.py:170-215) in the reference's arithmetic.
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


def _is_mse(policy) -> bool:
    return getattr(getattr(policy, "mode", None), "value", "absmax") == "mse"


def _check_policy(policy, fmt: int, mse: bool = False) -> None:
    """Policies the GPU path encodes; ``policy.mode`` is ignored by quantize_rtn, as in the
    reference (quantizers.py:247-255), and dispatched by ``quantize`` (:341-347)."""
    if policy is None:
        return
    if getattr(policy, "scale_fit", None) is not None:
        raise DataError("unsupported on GPU path: scale_fit (fitted E8M0 grid is not hardware E8M0)")


def _mx_four_thirds(policy) -> bool:
    return True if policy is None else bool(getattr(policy, "e8m0_four_thirds", True))


def as_device_matrix(X, device=None) -> torch.Tensor:
    """Validate like quantizers.py:95-101 (2-D, non-empty) and move to the GPU."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_23202_b200 needs a CUDA device (sm_100a); there is no CPU path")
    if not isinstance(X, torch.Tensor):
        X = torch.from_numpy(np.ascontiguousarray(np.asarray(X)))
    if X.dim() != 2 or X.shape[0] < 1 or X.shape[1] < 1:
        raise DataError("expected a non-empty 2-D matrix")
    if X.dtype not in _DT and X.dtype != torch.float64:
        X = X.to(torch.float64 if X.dtype in (torch.int64, torch.int32) else torch.float32)
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
        with torch.cuda.device(self.codes.device):
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
            with torch.cuda.device(X.device):
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
                   ts: torch.Tensor, scratch: torch.Tensor, *, four_thirds: bool = True,
                   static_ts: torch.Tensor | None = None) -> None:
    """Launch K1 on the current stream into caller-provided buffers (no allocation).
    ``four_thirds=False``: MXFP4 tensor scale 1.0 (ScalePolicy(e8m0_four_thirds=False));
    ``static_ts``: NVFP4 with a given device global scale (single pass)."""
    M, K = X.shape
    L = _lib.lib()
    opts = None
    if not four_thirds or static_ts is not None:
        if static_ts is not None and (static_ts.dtype != torch.float32 or static_ts.device != X.device):
            raise DataError("static tensor scale must be a float32 tensor on the input's device")
        opts = _lib.ActQuantOpts(int(four_thirds), _lib.ptr(static_ts) if static_ts is not None else None)
    with torch.cuda.device(X.device):   # launch on the tensors' device, not the current one
        _lib.check(L.mrfp4_act_quant_ex(_lib.ptr(X), _DT[X.dtype], M, K, X.stride(0), fmt, had_k,
                                        _lib.ptr(codes), _lib.ptr(sf), _lib.ptr(ts), _lib.ptr(scratch),
                                        _lib.ptr(scratch) + 16, 32,
                                        _lib.ctypes.byref(opts) if opts is not None else None,
                                        _lib.stream_ptr(torch, X.device)))


_SCRATCH: dict = {}


def stream_scratch(device) -> torch.Tensor:
    """K1 scratch shared by the stream-ordered calls that never read the status word
    (``quantized_linear(check=False)``): zeroed once; the NVFP4 workspace words re-arm
    themselves at the end of every launch, so no per-call zero-fill kernel is needed."""
    device = torch.device(device)
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    buf = _SCRATCH.get(key)
    if buf is None:
        buf = _SCRATCH[key] = torch.zeros(12, dtype=torch.int32, device=device)
    return buf


def alloc_result(M: int, K: int, fmt: int, had_k: int, device, scratch: torch.Tensor | None = None) -> GpuQuantResult:
    G = GROUP[fmt]
    sfb = _lib.lib().mrfp4_sf_bytes(M, K // G)
    return GpuQuantResult(
        fmt, M, K, had_k,
        torch.empty((M, K // 2), dtype=torch.uint8, device=device),
        torch.empty(sfb, dtype=torch.uint8, device=device),
        torch.empty(1, dtype=torch.float32, device=device),
        scratch if scratch is not None else torch.zeros(12, dtype=torch.int32, device=device))


def quantize_rtn(X, spec, policy=None, transform=None, *, check: bool = True,
                 static_tensor_scale=None) -> GpuQuantResult:
    """Round-to-nearest FP4 quantization with absmax scales, on the GPU.

    Drop-in for ``microfp.quantize_rtn`` (quantizers.py:247-255) for the MXFP4 /
    NVFP4 presets and Hadamard blocks 16/32/64/128 (or no transform), including
    ``ScalePolicy(e8m0_four_thirds=False)`` (quantizers.py:206-207) and float64 input.
    ``check=True`` (the reference behaviour) synchronizes to raise ``DataError`` on
    non-finite data; pass ``check=False`` to stay asynchronous and call
    ``.check()`` later.
    ``static_tensor_scale`` (NVFP4, not in the reference API): a precomputed global scale s_T
    (float or device float32 tensor) replacing the whole-tensor max --
    one pass, rows independent; codes are prepare_scales' with that s_global.
    """
    fmt = format_code(spec)
    _check_policy(policy, fmt)
    four_thirds = _mx_four_thirds(policy)
    had_k = hadamard_block(transform)
    X = as_device_matrix(X)
    M, K = X.shape
    G = GROUP[fmt]
    if K % G:                                                       # quantizers.py:106-107
        raise DataError(f"columns ({K}) not divisible by group size ({G})")
    if had_k and K % had_k:                                         # quantizers.py:108-111
        raise DataError(f"columns ({K}) not divisible by transform block ({had_k})")
    st = _static_ts(static_tensor_scale, fmt, X.device)
    if X.dtype == torch.float64:
        return _quantize_rtn_f64(X, fmt, had_k, four_thirds, st, check)
    res = alloc_result(M, K, fmt, had_k, X.device)
    act_quant_into(X, fmt, had_k, res.codes, res.sf, res.tensor_scale_dev, res.scratch,
                   four_thirds=four_thirds, static_ts=st)
    res.source = X
    if check:
        res.check()
    return res


def _static_ts(value, fmt: int, device) -> torch.Tensor | None:
    if value is None:
        return None
    if fmt != FMT_NVFP4:
        raise DataError("static_tensor_scale applies to NVFP4 only (MXFP4 has no global scale)")
    t = value if isinstance(value, torch.Tensor) else torch.tensor([float(value)], dtype=torch.float32)
    t = t.to(device=device, dtype=torch.float32).reshape(1)
    if not isinstance(value, torch.Tensor) and not (np.isfinite(float(value)) and float(value) > 0):
        raise DataError("static tensor scale must be finite and positive")
    return t


_FP4_MAG = (0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0)


def _quantize_rtn_f64(X: torch.Tensor, fmt: int, had_k: int, four_thirds: bool, static_ts, check: bool):
    """quantize_rtn of a float64 matrix in the reference's float64 arithmetic, on the device:
    apply_blockwise (mrfp4_rotate_f64, transforms.py:77-91), absmax / raw / s_T (quantizers.py:
    170-208), then the float64 encoder of the MSE pass run with the single candidate 1.0 --
    fp_scale_encode of raw / s_global and u = y / eff rounded onto E2M1 (quantizers.py:157-167,
    :211-215; formats.py:94-113, :220-262) -- and the metrics of quantizers.py:218-231."""
    if not bool(torch.isfinite(X).all()):                                  # quantizers.py:99-100
        if check:
            raise DataError("non-finite element")
    M, K = X.shape
    dev = X.device
    G = GROUP[fmt]
    ng = M * K // G
    L = _lib.lib()
    with torch.cuda.device(dev):
        stream = _lib.stream_ptr(torch, dev)
        Y = torch.empty((M, K), dtype=torch.float64, device=dev)
        _lib.check(L.mrfp4_rotate_f64(_lib.ptr(X), M, K, X.stride(0), had_k, _lib.ptr(Y), stream))
        B = Y.view(ng, G)
        absmax = B.abs().amax(dim=1)
        raw0 = torch.where(absmax == 0, torch.ones_like(absmax), absmax / 6.0).contiguous()
        if fmt == FMT_NVFP4:
            if static_ts is not None:
                s_global = float(static_ts.item())
            else:                                                          # quantizers.py:195-200
                top = float(absmax.max()) / 6.0
                s_global = float(np.float32(top / 448.0)) if top > 0 else 1.0
            ts = float(np.float32(s_global))
        else:
            s_global, ts = 1.0, float(np.float32(4.0 / 3.0)) if four_thirds else 1.0
        cand = torch.ones(1, dtype=torch.float64, device=dev)
        sc = torch.empty(ng, dtype=torch.uint8, device=dev)
        dec = torch.empty(ng, dtype=torch.float64, device=dev)
        gerr = torch.empty(ng, dtype=torch.float64, device=dev)
        res = alloc_result(M, K, fmt, had_k, dev)
        _lib.check(L.mrfp4_mse_pass(_lib.ptr(Y), ng, fmt, _lib.ptr(cand), 1, _lib.ptr(raw0), s_global, ts,
                                    _lib.ptr(sc), _lib.ptr(dec), _lib.ptr(gerr), _lib.ptr(res.codes),
                                    _lib.ptr(res.scratch), stream))
        _lib.check(L.mrfp4_sf_swizzle(_lib.ptr(sc), _lib.ptr(res.sf), M, K // G, stream))
        res.tensor_scale_dev.fill_(ts)
        # metrics (quantizers.py:218-231), rotated domain, float64
        x2 = float((Y * Y).sum())
        e2 = float(gerr.sum())
        arg = B.abs().argmax(dim=1, keepdim=True)                         # first maximum, as np.argmax
        top = B.gather(1, arg).squeeze(1)
        c = res.codes.view(ng, G // 2)
        nib = torch.stack((c & 15, c >> 4), dim=2).view(ng, G).gather(1, arg).squeeze(1).long()
        mag = torch.tensor(_FP4_MAG, dtype=torch.float64, device=dev)[nib & 7]
        q = torch.where((nib & 8) != 0, -mag, mag) * (ts * dec)
        t2 = top * top
        ratio = torch.where(t2 > 0, (top - q) ** 2 / torch.where(t2 > 0, t2, torch.ones_like(t2)),
                            torch.zeros_like(t2))
        res._metrics = (e2 / x2 if x2 > 0 else 0.0, float(ratio.mean()))
    if check:
        res.check()
    return res


def quantize(X, spec, policy=None, transform=None, *, check: bool = True) -> GpuQuantResult:
    """``microfp.quantize`` dispatch (quantizers.py:341-347): ScaleMode.MSE runs the MSE scale
    search (``mse_optimize_scales``) on the GPU, anything else is ``quantize_rtn``."""
    if _is_mse(policy):
        return mse_optimize_scales(X, spec, transform=transform, policy=policy, check=check)
    return quantize_rtn(X, spec, policy=policy, transform=transform, check=check)


MSE_SEARCH_MULTIPLIERS = np.linspace(0.50, 1.20, 128)   # quantizers.py:36-39
MSE_SEARCH_ROUNDS = 3
MSE_SEARCH_RTOL = 1e-12
_CHUNK_GROUPS = 2048


def rotate_f64(X: torch.Tensor, had_k: int) -> torch.Tensor:
    """apply_blockwise (transforms.py:77-91) in float64 on the GPU: the integer Hadamard sums
    are exact (cuBLAS DGEMM of +-1 against bf16 / fp16 / fp32 inputs), then one rounding by
    RN64(1 / RN64(sqrt(k))), the same y = RN64(S * c) the K1 kernels decide on."""
    if X.dtype == torch.float64:   # the reference's own order (mrfp4_rotate_f64)
        M, K = X.shape
        Y = torch.empty((M, K), dtype=torch.float64, device=X.device)
        with torch.cuda.device(X.device):
            _lib.check(_lib.lib().mrfp4_rotate_f64(_lib.ptr(X), M, K, X.stride(0), had_k, _lib.ptr(Y),
                                                   _lib.stream_ptr(torch, X.device)))
        return Y
    Xd = X.to(torch.float64)
    if not had_k:
        return Xd.contiguous()
    M, K = Xd.shape
    idx = torch.arange(had_k, device=X.device)
    par = torch.zeros((had_k, had_k), dtype=torch.int64, device=X.device)
    a = idx[:, None] & idx[None, :]
    while bool(a.any()):
        par ^= a & 1
        a = a >> 1
    H = (1 - 2 * par).to(torch.float64)
    return torch.matmul(Xd.view(M, K // had_k, had_k), H).mul_(1.0 / float(np.sqrt(had_k))).view(M, K)


_SEG_LIMIT = 16384   # numpy-recursion subtrees at most this long are summed on the GPU, one per thread


class _NpSum:
    """np.sum of a device float64 vector, bit-identical: numpy's pairwise recursion
    (umath pairwise_sum) is cut into subtrees of <= _SEG_LIMIT elements, each summed on the GPU
    by ``mrfp4_pairwise_sums`` with numpy's own recursion, and the subtree sums are added on
    the host in numpy's tree order."""

    def __init__(self, segments, device, tree=None):
        self.segments = segments
        self.tree = tree
        self.starts = torch.tensor([a for a, _ in segments], dtype=torch.int64, device=device)
        self.lens = torch.tensor([b for _, b in segments], dtype=torch.int64, device=device)
        self.out = torch.empty(len(segments), dtype=torch.float64, device=device)

    @classmethod
    def whole(cls, n: int, device):
        leaves = []

        def build(lo, m):
            if m <= _SEG_LIMIT:
                leaves.append((lo, m))
                return len(leaves) - 1
            m2 = m // 2
            m2 -= m2 % 8
            return (build(lo, m2), build(lo + m2, m - m2))

        tree = build(0, n)
        return cls(leaves, device, tree)

    @classmethod
    def chunks(cls, n: int, chunk: int, device):
        return cls([(lo, min(chunk, n - lo)) for lo in range(0, n, chunk)], device)

    def segment_sums(self, a: torch.Tensor) -> np.ndarray:
        _lib.check(_lib.lib().mrfp4_pairwise_sums(_lib.ptr(a), _lib.ptr(self.starts), _lib.ptr(self.lens),
                                                  len(self.segments), _lib.ptr(self.out),
                                                  _lib.stream_ptr(torch, a.device)))
        return self.out.cpu().numpy()

    def total(self, a: torch.Tensor) -> float:
        sums = self.segment_sums(a)

        def ev(node):
            return float(sums[node]) if isinstance(node, int) else ev(node[0]) + ev(node[1])

        return ev(self.tree)


def mse_optimize_scales(X, spec, transform=None, policy=None, *, check: bool = True) -> GpuQuantResult:
    """``quantize_rtn`` with MSE-optimised scales on the GPU (quantizers.py:330-337,
    ``optimize_group_scales`` :263-327).

    Same alternating search as the reference: a pass picks, per group, the best of the
    absmax scale and 128 multipliers in [0.5, 1.2] (each rounded through the scale codec;
    ties keep the earliest); for NVFP4 the tensor scale is then scanned over the same 128
    multipliers; at most 3 rounds, stopping at a relative improvement < 1e-12.  Group scores
    are computed by ``mrfp4_mse_pass`` / ``mrfp4_mse_group_err`` in float64 with numpy's
    summation order, and their totals are summed with numpy, so the decisions are the
    reference's.  Raises ``DataError`` where the reference does (non-finite input; a candidate
    scale that decodes to 0).

    MXFP4 (no tensor-scale scan) is "online": every round's pass repeats the first with the same
    s_global, so the reference's loop always stops after one repeat; one pass decides, with no
    host round trip -- rotate + absmax + one mrfp4_mse_pass on the stream (QuTLASS's fused MSE
    activation quantizer).  ``check=False`` then leaves the DataError conditions
    in the status word (``.check()``).  NVFP4's s_T scan needs the candidates' whole-tensor
    totals, which are summed in numpy's order on the host (offline weights)."""
    fmt = format_code(spec)
    _check_policy(policy, fmt, mse=True)
    had_k = hadamard_block(transform)
    X = as_device_matrix(X)
    M, K = X.shape
    G = GROUP[fmt]
    if K % G:
        raise DataError(f"columns ({K}) not divisible by group size ({G})")
    if had_k and K % had_k:
        raise DataError(f"columns ({K}) not divisible by transform block ({had_k})")
    is_global = fmt == FMT_NVFP4
    if is_global and not bool(torch.isfinite(X).all()):                    # quantizers.py:99-100
        raise DataError("non-finite element")
    dev = X.device
    L = _lib.lib()
    stream = _lib.stream_ptr(torch, dev)
    Y = rotate_f64(X, had_k)
    ng = M * K // G
    B = Y.view(ng, G)
    absmax = B.abs().amax(dim=1)
    raw0 = torch.where(absmax == 0, torch.ones_like(absmax), absmax / 6.0).contiguous()
    s_global, factor = 1.0, 1.0
    if is_global:                                                         # quantizers.py:195-200
        top = float(absmax.max()) / 6.0
        s_global = float(np.float32(top / 448.0)) if top > 0 else 1.0
    elif getattr(policy, "e8m0_four_thirds", True) if policy is not None else True:
        factor = 4.0 / 3.0
    cand_np = np.concatenate([[1.0], MSE_SEARCH_MULTIPLIERS])
    cand = torch.from_numpy(cand_np).to(dev)
    sc = torch.empty(ng, dtype=torch.uint8, device=dev)
    dec = torch.empty(ng, dtype=torch.float64, device=dev)
    gerr = torch.empty(ng, dtype=torch.float64, device=dev)
    gerr2 = torch.empty(ng, dtype=torch.float64, device=dev)
    codes = torch.empty((M, K // 2), dtype=torch.uint8, device=dev)
    scratch = torch.zeros(12, dtype=torch.int32, device=dev)
    status = _lib.ptr(scratch)

    chunk_sum = _NpSum.chunks(ng, _CHUNK_GROUPS, dev)
    whole_sum = _NpSum.whole(ng, dev)

    def pass_groups(sg: float) -> float:
        ts = float(np.float32(sg * factor))
        _lib.check(L.mrfp4_mse_pass(_lib.ptr(Y), ng, fmt, _lib.ptr(cand), len(cand_np), _lib.ptr(raw0), sg, ts,
                                    _lib.ptr(sc), _lib.ptr(dec), _lib.ptr(gerr), _lib.ptr(codes), status, stream))
        total = 0.0   # quantizers.py:292-301: float(errs[lo:hi].sum()) accumulated chunk by chunk
        for v in chunk_sum.segment_sums(gerr):
            total += float(v)
        return total

    def total_err(sg: float) -> float:
        ts = float(np.float32(sg * factor))
        _lib.check(L.mrfp4_mse_group_err(_lib.ptr(Y), ng, fmt, _lib.ptr(dec), ts, _lib.ptr(gerr2), status, stream))
        return whole_sum.total(gerr2)

    if not is_global:   # MXFP4: one pass decides (see above); no totals, no host round trip
        ts = float(np.float32(s_global * factor))
        _lib.check(L.mrfp4_mse_pass(_lib.ptr(Y), ng, fmt, _lib.ptr(cand), len(cand_np), _lib.ptr(raw0), s_global, ts,
                                    _lib.ptr(sc), _lib.ptr(dec), _lib.ptr(gerr), _lib.ptr(codes), status, stream))
        res = alloc_result(M, K, fmt, had_k, dev, scratch)
        res.codes = codes
        _lib.check(L.mrfp4_sf_swizzle(_lib.ptr(sc), _lib.ptr(res.sf), M, K // G, stream))
        res.tensor_scale_dev.fill_(ts)
        res.source = X
        if check:
            st = res.status
            if st & _lib.STATUS_SCALE_UNDERFLOW:
                raise DataError("non-finite element (a candidate group scale underflows the scale format)")
            if st & _lib.STATUS_NONFINITE:
                raise DataError("non-finite element")
        return res
    best_total = pass_groups(s_global)
    for _ in range(MSE_SEARCH_ROUNDS):
        if is_global:
            anchor, improved_to = s_global, best_total
            for m in cand_np[1:]:
                sg_c = float(np.float32(m * anchor))
                if sg_c > 0:
                    e = total_err(sg_c)
                    if e < improved_to:
                        improved_to, s_global = e, sg_c
        improved_to = pass_groups(s_global)
        if best_total - improved_to < MSE_SEARCH_RTOL * max(best_total, 1e-300):
            best_total = improved_to
            break
        best_total = improved_to
    st = int(scratch[0].item())
    if st & _lib.STATUS_SCALE_UNDERFLOW:
        raise DataError("non-finite element (a candidate group scale underflows the scale format)")
    if st & _lib.STATUS_NONFINITE:
        raise DataError("non-finite element")
    res = alloc_result(M, K, fmt, had_k, dev)
    res.codes.copy_(codes)
    _lib.check(L.mrfp4_sf_swizzle(_lib.ptr(sc), _lib.ptr(res.sf), M, K // G, stream))
    res.tensor_scale_dev.fill_(float(np.float32(s_global * factor)))
    res.source = X
    return res
