"""Column-parallel (N-sharded) quantized linear across the GPUs of one node (K4).

Each rank owns rows [r*N/P, (r+1)*N/P) of the prepared weight (``PackedWeight.shard``),
runs K1 on the full activation (replicated: deterministic, so every rank produces
identical codes and tensor scale) and K2 on its shard, then the bf16 output
shards are all-gathered -- the only exchange on the path.
The reference has no distributed code; its functions are pure and row-independent
(SPEC.md:116, :353).

Two gathers:
* ``gather_columns``: one NCCL ``all_gather_into_tensor`` of the [M, N/P] blocks (NVLink /
  NVSwitch) and a permute to [M, N].
* ``PeerOutputs``: every rank's full [M, N] output is a
  ``torch.distributed._symmetric_memory`` buffer, rendezvoused once; K2's epilogue stores each
  row segment of this rank's column block straight into all P ranks' buffers over NVLink
  (``mrfp4_gemm_peers``), tile by tile while the GEMM runs -- no separate collective, no
  permute.  Ordering is device-side: a symmetric-memory barrier (a signal-pad kernel on the
  stream, no host sync) before the GEMM -- no rank overwrites a peer's buffer while that peer
  may still be reading the previous result -- and one after it, once every rank's stores have
  landed.
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


class PeerOutputs:
    """Symmetric [M, N] bf16 output buffers of every rank of ``group`` (one per rank,
    rendezvoused once; collective: every rank must construct it).  ``peers[r]`` is rank r's
    buffer mapped into this process, ``local`` this rank's own."""

    def __init__(self, M: int, N: int, group=None, device=None):
        import torch.distributed._symmetric_memory as symm_mem
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if N % (self.world * 128):
            raise DataError(f"N={N} must split into multiples of 128 rows across {self.world} ranks")
        if self.world > 8:
            raise DataError("the fused gather stores to at most 8 ranks")
        self.M, self.N = M, N
        self.local = symm_mem.empty((M, N), dtype=torch.bfloat16, device=device)
        self.handle = symm_mem.rendezvous(self.local, self.group)
        self.peers = [self.handle.get_buffer(r, (M, N), torch.bfloat16) for r in range(self.world)]

    def barrier(self, channel: int = 0) -> None:
        """Device-side barrier over the group on the current stream (signal pads, no host sync)."""
        self.handle.barrier(channel=channel)


def quantized_linear_sharded(x: torch.Tensor, w_shard: PackedWeight, group=None, *,
                             out_dtype=torch.bfloat16, gather: bool = True, peer_outputs=None) -> torch.Tensor:
    """Per-rank K1 + K2 on the weight shard, then the output all-gather.

    ``peer_outputs``: a ``PeerOutputs`` -- K2 stores this rank's columns into every rank's
    symmetric buffer from its epilogue (no NCCL, device-side barriers); the returned tensor is
    this rank's full output, valid until the next call with the same buffers.  A list of
    peer-mapped [M, N] bf16 tensors (one per rank, e.g. from another IPC mechanism) is accepted
    too and is ordered with a host stream sync + ``dist.barrier``.  Default: NCCL all-gather."""
    if peer_outputs is not None:
        from .quantize import act_quant_into, alloc_result, as_device_matrix
        rank = dist.get_rank(group)
        x2 = as_device_matrix(x.reshape(-1, x.shape[-1]), w_shard.device)
        a = alloc_result(x2.shape[0], x2.shape[1], w_shard.fmt, w_shard.had_k, x2.device)
        act_quant_into(x2, w_shard.fmt, w_shard.had_k, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
        n = w_shard.N
        if isinstance(peer_outputs, PeerOutputs):
            po = peer_outputs
            if (po.M, po.N) != (x2.shape[0], n * po.world):
                raise DataError(f"peer buffers are [{po.M}, {po.N}], the output is [{x2.shape[0]}, {n * po.world}]")
            po.barrier(0)     # WAR: every peer is done with the previous result
            gemm_into_peers(a, w_shard, [p[:, po.rank * n:(po.rank + 1) * n] for p in po.peers])
            po.barrier(1)     # every rank's column block has landed in every buffer
            return po.local
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
    bf16 output, peer-mapped (``PeerOutputs``) or local.  The caller orders the ranks."""
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
    with torch.cuda.device(w_shard.device):
        _lib.check(_lib.lib().mrfp4_gemm_peers(
            _lib.ptr(a.codes), _lib.ptr(a.sf), _lib.ptr(a.tensor_scale_dev),
            _lib.ptr(w_shard.codes), _lib.ptr(w_shard.sf), _lib.ptr(w_shard.tensor_scale_dev),
            arr, len(outs), M, w_shard.N, w_shard.K, ldd, w_shard.fmt, _lib.stream_ptr(torch, outs[0].device)))
