"""N-sharded linear on real GPUs.

* world 1 on one GPU (always run): the NCCL path and the symmetric-memory fused-gather path
  (``PeerOutputs``: rendezvous, device-side barriers, K2 peer stores) through the same code a
  multi-GPU job runs, bit-identical to the unsharded ``quantized_linear`` and within the
  north-star tolerance of the oracle.
* world 2..8 over NCCL (one process per GPU; skipped unless >= 2 GPUs are visible): every rank's
  gathered output, for both gathers, equals the unsharded linear bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2509_23202_b200 as P
from paper_2509_23202_b200.sharded import PeerOutputs, quantized_linear_sharded

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(fmt, M=384, K=2048, N=2048, seed=3):
    rng = np.random.default_rng(seed)
    X = O.bf16_round(rng.standard_normal((M, K)))
    W = O.bf16_round(rng.standard_normal((N, K)) / np.sqrt(K))
    k = 32 if fmt == "mxfp4" else 16
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    return X, W, k, spec


def _run_rank(rank, world, port, fmt, q):
    try:
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                                device_id=dev)
        X, W, k, spec = _problem(fmt)
        x = torch.from_numpy(X).to(dev).bfloat16()
        w = P.quantize_weight(torch.from_numpy(W).to(dev).bfloat16(), spec, P.TransformSpec.hadamard(k))
        ref = P.quantized_linear(x, w)
        ws = w.shard(rank, world)
        y_nccl = quantized_linear_sharded(x, ws)
        ok = torch.equal(y_nccl, ref)
        try:
            po = PeerOutputs(x.shape[0], w.N, device=dev)
        except Exception as e:  # symmetric memory unavailable on this node
            po, note = None, repr(e)
        if po is not None:
            for _ in range(3):   # repeated calls: the device-side barriers order reuse of the buffers
                y_f = quantized_linear_sharded(x, ws, peer_outputs=po)
                ok &= torch.equal(y_f, ref)
            note = "fused"
        torch.cuda.synchronize()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok" if ok else "mismatch", note))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), ""))


@pytest.mark.parametrize("fmt", ["mxfp4", "nvfp4"])
def test_sharded_world1_nccl_and_fused_gather(fmt):
    """World 1 on this GPU: the multi-GPU code paths end to end, against the oracle too."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_run_rank, args=(0, 1, port, fmt, q))
    p.start()
    rank, status, note = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", (status, note)
    X, W, k, spec = _problem(fmt)
    # the unsharded linear itself vs the oracle (fp32 output)
    w = P.quantize_weight(torch.from_numpy(W).cuda().bfloat16(), spec, P.TransformSpec.hadamard(k))
    y = P.quantized_linear(torch.from_numpy(X).cuda().bfloat16(), w, out_dtype=torch.float32).cpu().numpy()
    ref = O.linear_reference(O.quantize_rtn(X, fmt, hadamard=k), O.quantize_rtn(W, fmt, hadamard=k))
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) <= 1e-5
    print(f"world 1 {fmt}: {note}")


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("fmt", ["mxfp4", "nvfp4"])
def test_sharded_multi_gpu_nccl_and_fused_gather(fmt):
    world = min(torch.cuda.device_count(), 8)
    while 2048 % (world * 128):
        world -= 1
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_run_rank, args=(r, world, port, fmt, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(s == "ok" for _, s, _ in res), res
