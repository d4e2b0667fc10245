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
                             out_dtype=torch.bfloat16, gather: bool = True) -> torch.Tensor:
    """Per-rank K1 + K2 on the weight shard, then NCCL all-gather of the output."""
    y = quantized_linear(x, w_shard, out_dtype=out_dtype)
    y2 = y.reshape(-1, w_shard.N)
    if not gather:
        return y
    full = gather_columns(y2, group)
    return full.reshape(*x.shape[:-1], full.shape[-1])
