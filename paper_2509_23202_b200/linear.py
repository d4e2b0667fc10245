"""Weight preparation (K3) and the quantized linear (K1 + K2).

The reference has no linear function: the paper's layer is
``Q(X H_k) Q(W H_k)^T``, i.e. ``dequantize(Aq) @ dequantize(Wq).T``
with ``Aq = quantize_rtn(X, spec, transform=H_k)`` online and ``Wq`` from
``quantize_rtn(W, ..., H_k)`` / ``mr_gptq`` offline
(/root/reference/pkg/src/microfp/formats.py:424-442, quantizers.py:247-255,
gptq.py:274-300).  Here:

* ``prepare_weight`` validates a reference ``MfpTensor`` (or ``QuantResult``) and
  uploads its codes unchanged (same nibble order) and its scale codes swizzled into
  the tensor-core layout (``mrfp4_sf_swizzle``).  Fitted E8M0 grids
  (``scale_fit``, quantizers.py:144-154) have no hardware encoding and are rejected.
* ``quantize_weight`` is the GPU RTN of a dense weight (bit-identical to
  ``quantize_rtn(W, spec, transform=H_k)``, transforms.py:94-100 rotation folded).
* ``quantized_linear`` runs K1 on the activations and K2 (tcgen05 block-scaled GEMM).
* ``quantized_linear_host`` is the same on host buffers, copies pipelined with compute.
"""

from __future__ import annotations

import dataclasses
import os

import numpy as np
import torch

from . import _lib
from .errors import DataError
from .formats import FMT_MXFP4 as FMT_MXFP4_CODE, FMT_NVFP4 as FMT_NVFP4_CODE, GROUP, format_code, spec_for
from .quantize import GpuQuantResult, act_quant_into, alloc_result, as_device_matrix, quantize_rtn, stream_scratch
from .transforms import hadamard_block, transform_for

_OUT = {torch.bfloat16: _lib.DT_BF16, torch.float32: _lib.DT_F32}


@dataclasses.dataclass
class PackedWeight:
    """A weight [N, K] in the GEMM's device layout."""

    fmt: int
    had_k: int
    N: int
    K: int
    codes: torch.Tensor             # uint8 [N, K/2]
    sf: torch.Tensor                # uint8 swizzled scales
    tensor_scale_dev: torch.Tensor  # float32 [1]

    @property
    def spec(self):
        return spec_for(self.fmt)

    @property
    def transform(self):
        return transform_for(self.had_k)

    @property
    def device(self):
        return self.codes.device

    def shard(self, rank: int, world: int) -> "PackedWeight":
        """Rows [rank*N/P, (rank+1)*N/P) of the weight (column-parallel linear)."""
        if self.N % (world * 128):
            raise DataError(f"N={self.N} must split into multiples of 128 rows across {world} ranks")
        n = self.N // world
        r0 = rank * n
        G = GROUP[self.fmt]
        cb = -(-(self.K // G) // 4)
        atoms = slice((r0 // 128) * cb * 512, ((r0 + n) // 128) * cb * 512)  # 128-row SF blocks are contiguous
        return PackedWeight(self.fmt, self.had_k, n, self.K, self.codes[r0:r0 + n].contiguous(),
                            self.sf[atoms].contiguous(), self.tensor_scale_dev.clone())


def _validate_gemm_k(K: int) -> None:
    if K % 64:
        raise DataError(f"unsupported on GPU path: K={K} must be a multiple of 64 for the FP4 GEMM")


def prepare_weight(w, device=None) -> PackedWeight:
    """MfpTensor / QuantResult / GpuQuantResult / MFPQ path -> PackedWeight on the GPU."""
    if isinstance(w, PackedWeight):
        return w
    if isinstance(w, GpuQuantResult):
        if getattr(w, "scale_fit", None) is not None:
            raise DataError("unsupported on GPU path: scale_fit weights (fitted E8M0 grid 2^(a*q+b) is not "
                            "hardware E8M0; quantize with absmax scales)")
        _validate_gemm_k(w.cols)
        # The clone is a plain stream-ordered copy, i.e. an ordering point outside the PDL chain:
        # the GEMM issues its weight loads before griddepcontrol.wait, so it must never become a
        # programmatic dependent of the K1 launch still writing this weight.
        with torch.cuda.device(w.codes.device):
            ts = w.tensor_scale_dev.clone()
        return PackedWeight(w.fmt, w.had_k, w.rows, w.cols, w.codes, w.sf, ts)
    if isinstance(w, (str, os.PathLike)):
        from .fileio import read_quant
        w, _perm = read_quant(w)  # the permutation section is informational (codes are un-permuted)
    if hasattr(w, "tensor") and not hasattr(w, "codes"):
        w = w.tensor  # reference QuantResult
    for attr in ("spec", "rows", "cols", "codes", "scale_codes", "tensor_scale"):
        if not hasattr(w, attr):
            raise DataError(f"prepare_weight: expected an MfpTensor-like object (missing {attr!r})")
    fmt = format_code(w.spec)
    if getattr(w, "scale_fit", None) is not None:
        raise DataError("unsupported on GPU path: scale_fit weights (fitted E8M0 grid 2^(a*q+b) is not "
                        "hardware E8M0; re-quantize with absmax scales, cli.py --scale-opt absmax)")
    had_k = hadamard_block(getattr(w, "transform", None))
    N, K = int(w.rows), int(w.cols)
    G = GROUP[fmt]
    _validate_gemm_k(K)
    codes = np.ascontiguousarray(np.asarray(w.codes, dtype=np.uint8).reshape(N, K // 2))
    sc = np.asarray(w.scale_codes)
    if sc.dtype.kind == "f":
        raise DataError("unsupported on GPU path: unquantized (float) scales")
    sc = np.ascontiguousarray(sc.astype(np.uint8).reshape(N, K // G))
    if fmt == 1 and sc.size and sc.max() > 126:
        raise DataError("reserved scale code in container")
    ts = float(w.tensor_scale)
    if not np.isfinite(ts) or ts <= 0:
        raise DataError("tensor_scale must be finite and positive")
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_23202_b200 needs a CUDA device (sm_100a); there is no CPU path")
    dev = torch.device(device or "cuda")
    d_codes = torch.from_numpy(codes).to(dev)
    d_sc = torch.from_numpy(sc).to(dev)
    d_sf = torch.empty(_lib.lib().mrfp4_sf_bytes(N, K // G), dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib().mrfp4_sf_swizzle(_lib.ptr(d_sc), _lib.ptr(d_sf), N, K // G,
                                           _lib.stream_ptr(torch, dev)))
    d_ts = torch.tensor([ts], dtype=torch.float32, device=dev)
    return PackedWeight(fmt, had_k, N, K, d_codes, d_sf, d_ts)


def quantize_weight(W, spec, transform=None, *, check: bool = True) -> PackedWeight:
    """GPU RTN of a dense weight with the rotation folded in (transforms.py:94-100)."""
    return prepare_weight(quantize_rtn(W, spec, transform=transform, check=check))


_WORKSPACE: dict = {}


def _gemm_workspace(device: torch.device, stream: int, nbytes: int):
    """GEMM scratch (split-K tile counters + fp32 partials) for eager calls: one zero-initialised,
    growing buffer per (device, stream), so stream-ordered reuse is safe (every call leaves
    the counter words zero again).  CUDA graphs must not use it (a later, larger request
    replaces -- frees -- the buffer a graph captured): ``GraphedLinear`` owns its workspace."""
    if nbytes == 0:
        return None
    key = (device.index, stream)
    buf = _WORKSPACE.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)  # split-K counters start at zero
        _WORKSPACE[key] = buf
    return buf


def gemm_workspace_bytes(M: int, w: PackedWeight) -> int:
    return int(_lib.lib().mrfp4_gemm_workspace(M, w.N, w.K, w.fmt))


def _check_out(out: torch.Tensor, M: int, w: PackedWeight) -> None:
    if not isinstance(out, torch.Tensor) or out.dtype not in _OUT:
        raise DataError("out must be a torch.bfloat16 or torch.float32 tensor")
    if out.device != w.device:
        raise DataError(f"out is on {out.device}, the weight on {w.device}")
    if out.dim() != 2 or tuple(out.shape) != (M, w.N):
        raise DataError(f"out must have shape ({M}, {w.N}), got {tuple(out.shape)}")
    if out.stride(1) != 1 or out.stride(0) < w.N:
        raise DataError("out must be row-major with unit column stride")


def gemm(a: GpuQuantResult, w: PackedWeight, out: torch.Tensor, ws: torch.Tensor | None = None) -> torch.Tensor:
    """K2 only: out[M, N] = a . w^T with both operands already quantized.  ``ws``: an explicit,
    zero-initialised split-K workspace of ``gemm_workspace_bytes`` bytes (CUDA graphs);
    default: the per-(device, stream) eager workspace."""
    if a.fmt != w.fmt or a.cols != w.K:
        raise DataError("activation / weight format or K mismatch")
    if a.codes.device != w.device:
        raise DataError(f"activation on {a.codes.device}, weight on {w.device}")
    _check_out(out, a.rows, w)
    L = _lib.lib()
    with torch.cuda.device(out.device):
        stream = _lib.stream_ptr(torch, out.device)
        nbytes = L.mrfp4_gemm_workspace(a.rows, w.N, w.K, w.fmt)
        if ws is None:
            ws = _gemm_workspace(out.device, stream, nbytes)
        elif ws.numel() < nbytes or ws.device != out.device:
            raise DataError(f"workspace needs {nbytes} bytes on {out.device}")
        _gemm_launch(L, a, w, out, ws, nbytes, stream)
    return out


def _gemm_launch(L, a, w, out, ws, nbytes, stream):
    _lib.check(L.mrfp4_gemm(
        _lib.ptr(a.codes), _lib.ptr(a.sf), _lib.ptr(a.tensor_scale_dev),
        _lib.ptr(w.codes), _lib.ptr(w.sf), _lib.ptr(w.tensor_scale_dev),
        _lib.ptr(out), _OUT[out.dtype], a.rows, w.N, w.K, out.stride(0), w.fmt,
        _lib.ptr(ws), nbytes, stream))


_DECODE = os.environ.get("MRFP4_DECODE", "1") != "0"   # A/B switch for the fused decode kernel
_IN = {torch.bfloat16: _lib.DT_BF16, torch.float16: _lib.DT_F16}


def decode_eligible(M: int, w: PackedWeight, x_dtype) -> bool:
    """Shapes the one-kernel decode linear (mrfp4_linear_decode) takes."""
    if not (_DECODE and 1 <= M <= 32 and w.K % 256 == 0 and w.N % 128 == 0
            and w.had_k in (0, 16, 32, 64, 128) and x_dtype in _IN):
        return False
    return int(_lib.lib().mrfp4_linear_decode_ctas(M, w.N, w.K)) > 0


def decode_workspace_bytes(M: int, w: PackedWeight) -> int:
    return int(_lib.lib().mrfp4_linear_decode_workspace(M, w.N, w.K))


def _linear_decode(x2: torch.Tensor, w: PackedWeight, out: torch.Tensor, ws, status) -> None:
    """K1 + K2 of a decode-sized linear in one launch (see include/mrfp4.h)."""
    M, K = x2.shape
    nbytes = decode_workspace_bytes(M, w)
    with torch.cuda.device(out.device):
        stream = _lib.stream_ptr(torch, out.device)
        if ws is None:
            ws = _gemm_workspace(out.device, ("dec", stream), nbytes)
        _lib.check(_lib.lib().mrfp4_linear_decode(
            _lib.ptr(x2), _IN[x2.dtype], M, K, w.fmt, w.had_k, _lib.ptr(w.codes), _lib.ptr(w.sf),
            _lib.ptr(w.tensor_scale_dev), w.N, _lib.ptr(out), _OUT[out.dtype], out.stride(0), _lib.ptr(ws), nbytes,
            _lib.ptr(status), stream))


def quantized_linear(x, w: PackedWeight, *, out_dtype=torch.bfloat16, out: torch.Tensor | None = None,
                     check: bool = False) -> torch.Tensor:
    """y = Q(x H_k) Q(W H_k)^T for x [..., K] (bf16/fp16/fp32), W prepared by prepare_weight."""
    if not isinstance(w, PackedWeight):
        w = prepare_weight(w)
    if out_dtype not in _OUT:
        raise DataError("out_dtype must be torch.bfloat16 or torch.float32")
    lead = tuple(x.shape[:-1]) if isinstance(x, torch.Tensor) else None
    x2 = as_device_matrix(x.reshape(-1, x.shape[-1]) if isinstance(x, torch.Tensor) else x, w.device)
    M, K = x2.shape
    if K != w.K:
        raise DataError(f"activation K={K} does not match weight K={w.K}")
    if decode_eligible(M, w, x2.dtype) and x2.is_contiguous():
        if out is None:
            out = torch.empty((M, w.N), dtype=out_dtype, device=x2.device)
        _check_out(out, M, w)
        status = torch.zeros(1, dtype=torch.int32, device=x2.device) if check else None
        _linear_decode(x2, w, out, None, status)
        if check and int(status.item()) & (_lib.STATUS_NONFINITE | _lib.STATUS_SCALE_UNDERFLOW):
            raise DataError("non-finite element")
        return out.reshape(*lead, w.N) if lead is not None and len(lead) != 1 else out
    # check=False never reads the status word: reuse the stream's scratch (no zero-fill launch)
    a = alloc_result(M, K, w.fmt, w.had_k, x2.device, None if check else stream_scratch(x2.device))
    act_quant_into(x2, w.fmt, w.had_k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    if check:
        a.check()
    if out is None:
        out = torch.empty((M, w.N), dtype=out_dtype, device=x2.device)
    gemm(a, w, out)
    return out.reshape(*lead, w.N) if lead is not None and len(lead) != 1 else out


class _HostPipe:
    """Per-(device, weight shape, chunk) device buffers and streams of quantized_linear_host."""

    def __init__(self, device, rows: int, K: int, N: int, fmt: int, had_k: int, x_dtype, out_dtype):
        self.x = [torch.empty((rows, K), dtype=x_dtype, device=device) for _ in range(2)]
        self.a = [alloc_result(rows, K, fmt, had_k, device) for _ in range(2)]
        self.y = [torch.empty((rows, N), dtype=out_dtype, device=device) for _ in range(2)]
        self.s_in = torch.cuda.Stream(device)
        self.s_comp = torch.cuda.Stream(device)
        self.s_out = torch.cuda.Stream(device)


_PIPES: dict = {}


def quantized_linear_host(x: torch.Tensor, w: PackedWeight, *, out: torch.Tensor | None = None,
                          out_dtype=torch.bfloat16, chunk_rows: int | None = None) -> torch.Tensor:
    """``quantized_linear`` on HOST buffers (the reference's CPU arrays in, arrays out).

    x is a CPU tensor [M, K] (bf16 / fp16 / fp32; pinned for asynchronous copies), the result
    is a CPU tensor [M, N] (``out`` if given, pinned).  Returns once the work is queued; the
    caller's current stream is ordered after the last device->host copy (synchronize it, or
    an event on it, before reading ``out``).

    MXFP4 scales are group-local, so rows are processed in chunks on three streams: the
    host->device copy of chunk i+1, K1+K2 of chunk i and the device->host copy of chunk i-1
    overlap (PCIe is full duplex), and the result is identical to one whole-matrix call.
    NVFP4's tensor scale is a max over the WHOLE activation (quantizers.py:198-200), so no
    row of it can be encoded before every row has arrived: NVFP4 runs copy -> K1+K2 -> copy.
    """
    if not isinstance(w, PackedWeight):
        w = prepare_weight(w)
    if x.device.type != "cpu" or x.dim() != 2:
        raise DataError("quantized_linear_host expects a 2-D CPU tensor")
    if out_dtype not in _OUT:
        raise DataError("out_dtype must be torch.bfloat16 or torch.float32")
    M, K = x.shape
    if K != w.K:
        raise DataError(f"activation K={K} does not match weight K={w.K}")
    if x.dtype not in (torch.bfloat16, torch.float16, torch.float32):
        x = x.float()
    x = x.contiguous()
    if not x.is_pinned():
        x = x.pin_memory()
    if out is None:
        out = torch.empty((M, w.N), dtype=out_dtype, pin_memory=True)
    elif out.shape != (M, w.N) or out.dtype not in _OUT or out.device.type != "cpu":
        raise DataError("out must be a CPU tensor [M, N] of bf16 / fp32")
    dev = w.device
    cur = torch.cuda.current_stream(dev)
    if w.fmt == FMT_NVFP4_CODE or M <= 128:
        xd = x.to(dev, non_blocking=True)
        y = quantized_linear(xd, w, out_dtype=out.dtype)
        out.copy_(y, non_blocking=True)
        return out
    rows = chunk_rows or max(128, ((M + 7) // 8 + 127) // 128 * 128)   # ~8 chunks
    key = (dev, rows, K, w.N, w.fmt, w.had_k, x.dtype, out.dtype)
    pipe = _PIPES.get(key)
    if pipe is None:
        pipe = _PIPES[key] = _HostPipe(dev, rows, K, w.N, w.fmt, w.had_k, x.dtype, out.dtype)
    start = torch.cuda.Event()
    start.record(cur)
    ev_in, ev_comp, ev_out = {}, {}, {}
    for i, r0 in enumerate(range(0, M, rows)):
        r1 = min(M, r0 + rows)
        n = r1 - r0
        b = i & 1
        with torch.cuda.stream(pipe.s_in):
            pipe.s_in.wait_event(start)
            if i >= 2:
                pipe.s_in.wait_event(ev_comp[i - 2])       # K1 of chunk i-2 has read x[b]
            pipe.x[b][:n].copy_(x[r0:r1], non_blocking=True)
            ev_in[i] = torch.cuda.Event()
            ev_in[i].record(pipe.s_in)
        with torch.cuda.stream(pipe.s_comp):
            pipe.s_comp.wait_event(ev_in[i])
            if i >= 2:
                pipe.s_comp.wait_event(ev_out[i - 2])      # y[b] of chunk i-2 copied out
            a = pipe.a[b]
            if n != rows:
                a = alloc_result(n, K, w.fmt, w.had_k, dev)
            act_quant_into(pipe.x[b][:n], w.fmt, w.had_k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
            gemm(a, w, pipe.y[b][:n])
            ev_comp[i] = torch.cuda.Event()
            ev_comp[i].record(pipe.s_comp)
        with torch.cuda.stream(pipe.s_out):
            pipe.s_out.wait_event(ev_comp[i])
            out[r0:r1].copy_(pipe.y[b][:n], non_blocking=True)
            ev_out[i] = torch.cuda.Event()
            ev_out[i].record(pipe.s_out)
    cur.wait_event(ev_out[max(ev_out)])
    cur.wait_event(ev_comp[max(ev_comp)])
    return out


def quantized_linear_requant(x, w: PackedWeight, next_transform=None, *, next_spec=None, next_tensor_scale=None,
                             keep_output: bool = False, check: bool = False):
    """``quantized_linear`` whose bf16 output is quantized for the NEXT layer in K2's epilogue
    (SURVEY.md 8(f) row f4): returns the GpuQuantResult that
    ``quantize_rtn(y, next_spec, transform=next_transform)`` would return for
    y = quantized_linear(x, w) -- bit-identical -- without writing y to HBM and reading it back
    (``keep_output=True`` also returns y).
    next_spec: FormatSpec.mxfp4() (default), or FormatSpec.nvfp4() with ``next_tensor_scale`` --
    a static global scale s_T (float or device float32 tensor), i.e.
    ``quantize_rtn(y, nvfp4, transform, static_tensor_scale=s_T)``: a whole-y s_T (quantizers.py:
    195-200) needs all of y before any group is encoded, so it cannot be fused.
    next_transform: None or a Hadamard block of 16 / 32 / 64 / 128."""
    if not isinstance(w, PackedWeight):
        w = prepare_weight(w)
    nfmt = FMT_MXFP4_CODE if next_spec is None else format_code(next_spec)
    st = None
    if nfmt == FMT_NVFP4_CODE:
        if next_tensor_scale is None:
            raise DataError("unsupported on GPU path: a fused NVFP4 requant needs a static next_tensor_scale")
        from .quantize import _static_ts
        st = _static_ts(next_tensor_scale, nfmt, w.device)
    elif next_tensor_scale is not None:
        raise DataError("next_tensor_scale applies to an NVFP4 next layer only")
    x2 = as_device_matrix(x, w.device)
    M, K = x2.shape
    if K != w.K:
        raise DataError(f"activation K={K} does not match weight K={w.K}")
    hk = hadamard_block(next_transform)
    a = alloc_result(M, K, w.fmt, w.had_k, x2.device)
    act_quant_into(x2, w.fmt, w.had_k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
    res = alloc_result(M, w.N, nfmt, hk, x2.device)
    y = torch.empty((M, w.N), dtype=torch.bfloat16, device=x2.device) if keep_output else None
    L = _lib.lib()
    with torch.cuda.device(x2.device):
        _lib.check(L.mrfp4_gemm_quant_next_ex(
            _lib.ptr(a.codes), _lib.ptr(a.sf), _lib.ptr(a.tensor_scale_dev),
            _lib.ptr(w.codes), _lib.ptr(w.sf), _lib.ptr(w.tensor_scale_dev),
            _lib.ptr(y) if y is not None else None, w.N, M, w.N, K, w.fmt, nfmt, hk, _lib.ptr(st),
            _lib.ptr(res.codes), _lib.ptr(res.sf), _lib.ptr(res.tensor_scale_dev), _lib.ptr(res.scratch),
            _lib.stream_ptr(torch, x2.device)))
    if check:
        res.check()
    return (res, y) if keep_output else res


class GraphedLinear:
    """``quantized_linear`` for one fixed batch size, captured once into a CUDA graph.

    Decode-sized layers are launch-bound: K1, K2 (and the split-K reduce) cost a few
    microseconds of GPU time each but tens of microseconds of host work per call through
    Python.  ``GraphedLinear(w, M)`` records the whole layer (static input / output buffers,
    PDL edges kept) and ``__call__`` replays it: one graph launch per layer call.
    """

    def __init__(self, w: PackedWeight, M: int, *, x_dtype=torch.bfloat16, out_dtype=torch.bfloat16):
        if out_dtype not in _OUT:
            raise DataError("out_dtype must be torch.bfloat16 or torch.float32")
        self.w = w
        dev = w.device
        self.x = torch.zeros((M, w.K), dtype=x_dtype, device=dev)
        self.y = torch.empty((M, w.N), dtype=out_dtype, device=dev)
        self.a = alloc_result(M, w.K, w.fmt, w.had_k, dev)
        # The graph captures raw pointers: it owns its split-K workspace (zeroed once; every
        # replay leaves the counters zero again) instead of borrowing the shared eager one.
        self.decode = decode_eligible(M, w, x_dtype)
        nbytes = decode_workspace_bytes(M, w) if self.decode else gemm_workspace_bytes(M, w)
        self.ws = torch.zeros(max(nbytes, 1), dtype=torch.uint8, device=dev)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(2):   # warm-up: kernel attributes, tensor maps, GEMM workspace
                self._run()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=side):
            self._run()
        torch.cuda.synchronize(dev)

    def _run(self):
        if self.decode:
            _linear_decode(self.x, self.w, self.y, self.ws, None)
            return
        act_quant_into(self.x, self.w.fmt, self.w.had_k, self.a.codes, self.a.sf, self.a.tensor_scale_dev,
                       self.a.scratch)
        gemm(self.a, self.w, self.y, ws=self.ws)

    def __call__(self, x: torch.Tensor | None = None) -> torch.Tensor:
        """Replay on the current stream; ``x`` (same shape) is copied into the static input first.
        Returns the static output buffer (overwritten by the next call)."""
        if x is not None:
            self.x.copy_(x, non_blocking=True)
        self.graph.replay()
        return self.y
