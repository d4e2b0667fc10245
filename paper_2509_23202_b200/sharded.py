"""Column-parallel (N-sharded) quantized linear across the GPUs of one node (K4).

Each rank owns rows [r*N/P, (r+1)*N/P) of the prepared weight (``PackedWeight.shard``),
runs K1 on the full activation (replicated: deterministic, so every rank produces
identical codes and tensor scale) and K2 on its shard, then the bf16 output
shards are all-gathered over NCCL (NVLink / NVSwitch) -- the only collective on
the path.  The reference has no distributed code; its
functions are pure and row-independent.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .errors import DataError
from .linear import PackedWeight, quantized_linear


def shard_rows(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """[start, stop) of this rank's output columns; shards are 128-row aligned."""
    if n_rows % (world * 128):
        raise DataError(f"N={n_rows} must split into multiples of 128 rows across {world} ranks")
    n = n_rows // world
    return rank * n, (rank + 1) * n


def gather_columns(y_shard: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather [M, N/P] shards from every rank into the full [M, N] output."""
    world = dist.get_world_size(group)
    if world == 1:
        return y_shard
    M, n = y_shard.shape
    buf = torch.empty((world * M, n), dtype=y_shard.dtype, device=y_shard.device)  # rank-major [P*M, N/P]
    dist.all_gather_into_tensor(buf, y_shard.contiguous(), group=group)
    return buf.view(world, M, n).permute(1, 0, 2).reshape(M, world * n)


def quantized_linear_sharded(x: torch.Tensor, w_shard: PackedWeight, group=None, *,
                             out_dtype=torch.bfloat16, gather: bool = True, peer_outputs=None) -> torch.Tensor:
    """Per-rank K1 + K2 on the weight shard, then NCCL all-gather of the output.

    ``peer_outputs``: every rank's full [M, N] bf16 output buffer mapped into this process
    (symmetric memory over NVLink), indexed by rank.  K2 then stores this rank's columns into all
    of them from its epilogue (``gemm_into_peers``) instead of running the NCCL all-gather; the
    ranks synchronize before the result is returned.  (Emulation-tested on one GPU only.)"""
    if peer_outputs is not None:
        from .quantize import act_quant_into, alloc_result, as_device_matrix
        rank = dist.get_rank(group)
        x2 = as_device_matrix(x.reshape(-1, x.shape[-1]), w_shard.device)
        a = alloc_result(x2.shape[0], x2.shape[1], w_shard.fmt, w_shard.had_k, x2.device)
        act_quant_into(x2, w_shard.fmt, w_shard.had_k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
        n = w_shard.N
        # write-after-read: no rank may store into a peer's output while that peer may still be
        # consuming the previous call's result from it
        torch.cuda.current_stream(x2.device).synchronize()
        dist.barrier(group)
        gemm_into_peers(a, w_shard, [po[:, rank * n:(rank + 1) * n] for po in peer_outputs])
        torch.cuda.current_stream(x2.device).synchronize()
        dist.barrier(group)
        return peer_outputs[rank]
    y = quantized_linear(x, w_shard, out_dtype=out_dtype)
    y2 = y.reshape(-1, w_shard.N)
    if not gather:
        return y
    full = gather_columns(y2, group)
    return full.reshape(*x.shape[:-1], full.shape[-1])


def gemm_into_peers(a, w_shard: PackedWeight, outs: list) -> None:
    """K2 of this rank's weight shard with the output all-gather fused into the epilogue
    (``mrfp4_gemm_peers``): every output row segment is stored into each
    tensor of ``outs`` -- this rank's [M, N/P] column block inside every rank's full [M, N]
    bf16 output, peer-mapped (e.g. ``torch.distributed._symmetric_memory`` buffers over
    NVLink) or local.  The caller synchronizes the ranks before reading."""
    import ctypes

    from . import _lib
    if not 1 <= len(outs) <= 8:
        raise DataError("1..8 destinations")
    M = a.rows
    ldd = outs[0].stride(0)
    for o in outs:
        if o.dtype != torch.bfloat16 or tuple(o.shape) != (M, w_shard.N) or o.stride() != (ldd, 1):
            raise DataError("destinations must be bf16 [M, N/P] views with one common row stride")
    arr = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    _lib.check(_lib.lib().mrfp4_gemm_peers(
        _lib.ptr(a.codes), _lib.ptr(a.sf), _lib.ptr(a.tensor_scale_dev),
        _lib.ptr(w_shard.codes), _lib.ptr(w_shard.sf), _lib.ptr(w_shard.tensor_scale_dev),
        arr, len(outs), M, w_shard.N, w_shard.K, ldd, w_shard.fmt, _lib.stream_ptr(torch, outs[0].device)))
