"""Host logic of the N-sharded (column-parallel) linear, world_size 2 over gloo on CPU.

The sharded path (paper_2509_23202_b200/sharded.py) is:
each rank owns rows [r*N/P, (r+1)*N/P) of the prepared weight, computes its
[M, N/P] output block, and one all-gather assembles [M, N].  These tests check,
without a GPU, that (1) ``PackedWeight.shard`` slices codes and the swizzled
scale-factor atoms so every shard is a self-consistent weight of N/P rows, and
(2) ``gather_columns`` reassembles the per-rank blocks into exactly the
unsharded oracle output (dequantize(A) @ dequantize(W).T, formats.py:424-442), and (3)
``quantized_linear_sharded``'s host flow reproduces it with the per-rank GPU linear replaced by
the oracle's block (the GPU path itself: tests/test_gpu_multi.py).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2509_23202_b200.errors import DataError
from paper_2509_23202_b200.formats import FMT_MXFP4, FMT_NVFP4
from paper_2509_23202_b200.linear import PackedWeight
from paper_2509_23202_b200.sharded import gather_columns, shard_rows

M, N, K = 24, 512, 256


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _weight(fmt_name: str):
    rng = np.random.default_rng(7)
    W = O.bf16_round(rng.standard_normal((N, K)) / 16)
    Wq = O.quantize_rtn(W, fmt_name, hadamard=32 if fmt_name == "mxfp4" else 16)
    pw = PackedWeight(FMT_MXFP4 if fmt_name == "mxfp4" else FMT_NVFP4, Wq.hadamard or 0, N, K,
                      torch.from_numpy(Wq.codes.copy()),
                      torch.from_numpy(O.sf_swizzle(Wq.scale_codes.reshape(N, -1))),
                      torch.tensor([Wq.tensor_scale], dtype=torch.float32))
    return Wq, pw


def _worker(rank: int, world: int, port: int, fmt_name: str, q):
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        Wq, pw = _weight(fmt_name)
        G = 32 if fmt_name == "mxfp4" else 16
        lo, hi = shard_rows(N, rank, world)
        sh = pw.shard(rank, world)
        # (1) the shard is the weight's row slice, scale factors included
        assert sh.N == hi - lo and sh.K == K
        assert np.array_equal(sh.codes.numpy(), Wq.codes[lo:hi])
        sf_rows = O.sf_unswizzle(sh.sf.numpy(), hi - lo, K // G)
        assert np.array_equal(sf_rows, Wq.scale_codes.reshape(N, -1)[lo:hi])
        assert float(sh.tensor_scale_dev[0]) == float(np.float32(Wq.tensor_scale))
        # (2) per-rank block -> all-gather == unsharded output
        rng = np.random.default_rng(11)
        X = O.bf16_round(rng.standard_normal((M, K)))
        Aq = O.quantize_rtn(X, fmt_name, hadamard=Wq.hadamard)
        y_full = O.linear_reference(Aq, Wq).astype(np.float32)
        y_blk = torch.from_numpy(np.ascontiguousarray(y_full[:, lo:hi]))
        y = gather_columns(y_blk, None)
        assert y.shape == (M, N)
        assert np.array_equal(y.numpy(), y_full)
        # (3) quantized_linear_sharded's host flow (leading dims, per-rank block, gather, reshape)
        # with the per-rank GPU linear replaced, for this CPU test only, by the oracle's block
        import paper_2509_23202_b200.sharded as S

        def block_linear(x, w_shard, out_dtype=torch.bfloat16):
            assert w_shard.N == hi - lo and tuple(x.shape[-1:]) == (K,)
            return torch.from_numpy(np.ascontiguousarray(y_full[:, lo:hi])).reshape(*x.shape[:-1], hi - lo)

        real = S.quantized_linear
        S.quantized_linear = block_linear
        try:
            x3 = torch.from_numpy(X.astype(np.float32)).reshape(2, M // 2, K)
            y3 = S.quantized_linear_sharded(x3, sh)
        finally:
            S.quantized_linear = real
        assert tuple(y3.shape) == (2, M // 2, N)
        assert np.array_equal(y3.reshape(M, N).numpy(), y_full)
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("fmt_name", ["mxfp4", "nvfp4"])
def test_sharded_linear_world2_gloo(fmt_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, fmt_name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_shard_rows_alignment():
    assert shard_rows(53248, 3, 8) == (3 * 6656, 4 * 6656)   # config 4: 6656 = 52 * 128
    with pytest.raises(DataError):
        shard_rows(4096 + 64, 0, 2)
