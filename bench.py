#!/usr/bin/env python
"""Benchmark of the MR-GPTQ FP4 quantized-linear hot path on B200 (driver contract).

One *step* = one pass of the hot path over one batch: K1 (online Hadamard rotate +
FP4 quantize of the activations, CUDA) then K2 (tcgen05 block-scaled FP4 GEMM
against RTN weights prepared once).  Default workload = BASELINE.json configs[1]:
Llama-3-8B MLP down_proj, K=14336 -> N=4096, 2048 tokens, MXFP4 + Hadamard-32.

Reported (one JSON line from rank 0):
  value / ms_per_step   FP4-linear TFLOP/s = 2*M*N*K / t_step, t_step = CUDA events around K1+K2
                        (back to back, PDL overlaps K2's prologue with K1's tail), inputs resident
                        in HBM, L2 flushed between steps: a 256 MiB memset, then a 256 MiB read
                        sweep of a second buffer so the flush's dirty lines are written back
                        outside the timed region
  e2e                   same metric through the public API (quantized_linear) with the
                        activations copied from pinned host memory and Y read back per step
  roofline              dominant kernel (K2) vs 4x the measured bf16 peak; K1 vs measured HBM
  cpu_baseline          the CPU oracle (numpy port of the reference) on a bounded sample
  extras                cuBLAS-bf16 time of the same layer and the layer speedup over it,
                        rot+quant GB/s, clocks sampled during the timed region
--impl reference times the stock reference (microfp staged into oracle/_ref by oracle/make_ref.py;
the numpy port when absent) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (workload, M, K, N, fmt, hadamard)
    "c1": ("llama3-8b mlp.down_proj 14336->4096, 2048 tokens, MXFP4+H32", 2048, 14336, 4096, "mxfp4", 32),
    "c0": ("llama3-8b attn.q_proj 4096->4096, 16 tokens, NVFP4+H16", 16, 4096, 4096, "nvfp4", 16),
    "c0-up": ("llama3-8b mlp.up_proj 4096->14336, 16 tokens, NVFP4+H16", 16, 4096, 14336, "nvfp4", 16),
    "c2-up-nv": ("llama3-70b mlp.up 8192->28672, 2048 tokens, NVFP4+H16", 2048, 8192, 28672, "nvfp4", 16),
    "c2-down-mx": ("llama3-70b mlp.down 28672->8192, 2048 tokens, MXFP4+H32", 2048, 28672, 8192, "mxfp4", 32),
    "c2-up-mx": ("llama3-70b mlp.up 8192->28672, 2048 tokens, MXFP4+H32", 2048, 8192, 28672, "mxfp4", 32),
    "c2-down-nv": ("llama3-70b mlp.down 28672->8192, 2048 tokens, NVFP4+H16", 2048, 28672, 8192, "nvfp4", 16),
    "c3-gateup": ("qwen3-32b mlp.gate_up 5120->51200, 2048 tokens, NVFP4+H128", 2048, 5120, 51200, "nvfp4", 128),
    "c4": ("llama3-405b-shaped mlp 16384->53248, 8192 tokens, NVFP4+H16", 8192, 16384, 53248, "nvfp4", 16),
}
METRIC = "FP4 linear TFLOPS & speedup vs BF16 at Llama-3 shapes; rot+quant HBM GB/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", 0)), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self, keep_busy=None):
        """Start sampling and return once the first sample is in (nvidia-smi takes ~0.1-0.5 s to
        come up; a timed region shorter than that would otherwise see no sample).  keep_busy()
        is called meanwhile so the GPU stays under the benchmark's load."""
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "20",
                 "-i", str(self.dev)], stdout=self.fh, stderr=subprocess.DEVNULL)
            t0 = time.time()
            while time.time() - t0 < 5.0 and os.path.getsize(self.path) == 0:
                if keep_busy is not None:
                    keep_busy()
                else:
                    time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


class stdout_to_stderr:
    """Route file descriptor 1 to 2 for a block (C-level library prints included)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False


# ----------------------------------------------------------------------------- CPU arms
def load_reference():
    """The stock reference package staged into oracle/_ref by oracle/make_ref.py, or None."""
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "microfp")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import microfp
    return microfp


def blas_threads() -> str:
    try:
        from threadpoolctl import threadpool_info
        return ", ".join(f"{d['internal_api']} {d['num_threads']} threads" for d in threadpool_info())
    except Exception:  # noqa: BLE001
        return "unknown"


class CpuArm:
    """One CPU quantized-linear step on a sample of the workload's token rows: the reference's
    own quantize_rtn(X, spec, transform) -> dequantize -> float64 matmul with the dequantized
    weight (kind "reference"), or the numpy port when oracle/_ref is absent (kind "port")."""

    def __init__(self, K, N, fmt, had, seed=1234):
        import numpy as np
        import oracle as O
        self.mf = load_reference()
        self.kind = "reference" if self.mf is not None else "port"
        self.fmt, self.had, self.K = fmt, had, K
        self.rng = np.random.default_rng(seed)
        W = O.bf16_round(self.rng.standard_normal((N, K), dtype=np.float32) / np.sqrt(K))
        if self.mf is not None:
            self.spec = self.mf.FormatSpec.mxfp4() if fmt == "mxfp4" else self.mf.FormatSpec.nvfp4()
            self.tr = self.mf.TransformSpec.hadamard(had) if had else None
            self.Wdeq = self.mf.dequantize(self.mf.quantize_rtn(W, self.spec, transform=self.tr).tensor)
        else:
            self.Wdeq = O.dequantize_f32(O.quantize_rtn_parallel(W, fmt, had))

    def inputs(self, rows):
        import numpy as np
        import oracle as O
        return O.bf16_round(self.rng.standard_normal((rows, self.K), dtype=np.float32))

    def step(self, X):
        if self.mf is not None:
            q = self.mf.quantize_rtn(X, self.spec, transform=self.tr)
            return self.mf.dequantize(q.tensor) @ self.Wdeq.T
        import oracle as O
        return O.dequantize_f32(O.quantize_rtn_parallel(X, self.fmt, self.had)) @ self.Wdeq.T

    def rows_for(self, seconds, cap):
        """Token rows per step so that one step takes about `seconds`."""
        import time as _t
        X = self.inputs(4)
        self.step(X)
        t0 = _t.perf_counter()
        self.step(X)
        per_row = (_t.perf_counter() - t0) / 4
        return int(max(1, min(cap, round(seconds / max(per_row, 1e-9)))))


def run_reference(args, cfg, rank):
    """--impl reference: the reference's own CPU implementation of the path (oracle/_ref, the
    stock microfp package), each step a bounded sample of the workload's token rows sized so the
    whole --warmup W --steps K run takes about two minutes; rank 0 only."""
    if rank != 0:
        return
    name, M, K, N, fmt, had = cfg
    arm = CpuArm(K, N, fmt, had)
    rows = arm.rows_for(min(2.0, 120.0 / (args.steps + args.warmup)), M)
    X = arm.inputs(rows)
    for _ in range(args.warmup):
        arm.step(X)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        arm.step(X)
    dt = (time.perf_counter() - t0) / args.steps
    tflops = 2.0 * rows * N * K / dt / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": tflops, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (bf16 N(0,1) acts, N(0,1/K) weights)",
        "config": {"workload": name, "M": M, "K": K, "N": N, "format": fmt, "hadamard": had},
        "cpu_baseline": {"value": tflops, "unit": "TFLOP/s", "cores": len(os.sched_getaffinity(0)),
                         "kind": arm.kind, "blas": blas_threads(),
                         "sample": f"{rows} of the {M} token rows per step, full K and N: quantize_rtn + "
                                   f"dequantize + float64 matmul ({'stock microfp' if arm.mf else 'numpy port'})"},
        "e2e": {"value": tflops, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sustained", action="store_true")
    ap.add_argument("--no-comparators", action="store_true")
    ap.add_argument("--M", type=int, default=0, help="override the config's token count (sweeps)")
    ap.add_argument("--gather", default="auto", choices=["auto", "nccl", "fused"],
                    help="N-sharded output gather: NCCL all-gather, the K2 epilogue's peer stores into "
                         "symmetric memory, or (auto, N > 1) both, reporting the faster")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.M:
        cfg = (cfg[0].rsplit(",", 2)[0] + f", {args.M} tokens," + cfg[0].rsplit(",", 1)[1],
               args.M) + tuple(cfg[2:])

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2509_23202_b200 as P
    from paper_2509_23202_b200.quantize import act_quant_into, alloc_result
    from paper_2509_23202_b200.sharded import PeerOutputs, gather_columns, gemm_into_peers

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or args.gather != "auto"
    if sharded:
        dist.init_process_group("nccl", device_id=dev)

    name, M, K, N, fmt, had = cfg
    spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
    tr = P.TransformSpec.hadamard(had)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    x = torch.randn((M, K), generator=g, device=dev, dtype=torch.float32).bfloat16()
    g.manual_seed(4321)
    w_dense = (torch.randn((N, K), generator=g, device=dev, dtype=torch.float32) / K ** 0.5).bfloat16()
    w_full = P.quantize_weight(w_dense, spec, tr)            # GPU RTN == reference quantize_rtn(W, ..., H)
    w = w_full.shard(rank, world) if sharded else w_full
    a = alloc_result(M, K, w.fmt, had, dev)
    y = torch.empty((M, w.N), dtype=torch.bfloat16, device=dev)
    flush_w = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
    flush_r = torch.ones(64 * 2 ** 20, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def flush_l2():
        flush_w.zero_()                    # write a buffer larger than L2 (126 MB) ...
        flush_r.sum(dtype=torch.int32)     # ... then read another: L2 left clean, none of our data

    # K1 (one launch for both formats) + K2 (split-K for small M reduces inside K2)
    launches_per_step = 2

    # N-sharded: time-to-gathered-output, through the NCCL all-gather or the fused peer-store gather
    gathers = []
    if sharded:
        gathers = ["nccl", "fused"] if args.gather == "auto" else [args.gather]
    po = None
    if "fused" in gathers:
        try:
            po = PeerOutputs(M, N, device=dev)
        except Exception as e:  # symmetric memory unavailable: decided collectively below
            print(f"fused gather unavailable: {e!r}", file=sys.stderr)
            po = None
    cols = slice(rank * w.N, (rank + 1) * w.N)

    # Decode-sized layers (M <= 32) run as ONE kernel: the act-quant inside the GEMM CTAs
    # (mrfp4_linear_decode), which is what quantized_linear launches for them.
    from paper_2509_23202_b200.linear import _linear_decode, decode_eligible, decode_workspace_bytes
    fused_decode = not sharded and decode_eligible(M, w, x.dtype) and os.environ.get("MRFP4_DECODE", "1") != "0"
    if fused_decode:
        launches_per_step = 1
        dws = torch.zeros(max(decode_workspace_bytes(M, w), 1), dtype=torch.uint8, device=dev)

    def step_nccl():
        if fused_decode:
            _linear_decode(x, w, y, dws, None)
            return y
        act_quant_into(x, w.fmt, had, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
        P.gemm(a, w, y)
        if sharded:
            return gather_columns(y, None)
        return y

    def step_fused():
        act_quant_into(x, w.fmt, had, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
        po.barrier(0)
        gemm_into_peers(a, w, [pp[:, cols] for pp in po.peers])
        po.barrier(1)

    step = step_nccl

    # The fused gather is checked against the NCCL one on this node before it is timed, and the
    # decision to keep it is collective (a rank that would skip it alone would hang the others).
    if sharded and "fused" in gathers:
        ok = po is not None
        if ok:
            try:
                ref = step_nccl().clone()
                step_fused()
                torch.cuda.synchronize(dev)
                ok = bool(torch.equal(po.local, ref))
            except Exception as e:  # noqa: BLE001
                print(f"fused gather failed its check: {e!r}", file=sys.stderr)
                ok = False
        flag = torch.tensor([1 if ok else 0], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not int(flag.item()):
            print("fused gather disabled on every rank (unavailable or mismatching)", file=sys.stderr)
            gathers = [gg for gg in gathers if gg != "fused"] or ["nccl"]

    def barrier():
        if sharded:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # ---------------- device-timed hot path (L2 flushed before every step)
    def timed(fn, n):
        """Per-iteration device times (s) of fn, CUDA events on the launching stream."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for e0, e1 in ev:
            flush_l2()
            e0.record(stream)
            fn()
            e1.record(stream)
        return ev

    variants = {gg: (step_fused if gg == "fused" else step_nccl) for gg in gathers} or {"none": step_nccl}
    for fn in variants.values():
        for _ in range(args.warmup):
            flush_l2()
            fn()
        barrier()

    def busy():   # local work only (no collective: ranks may loop a different number of times)
        for _ in range(10):
            flush_l2()
            act_quant_into(x, w.fmt, had, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
            P.gemm(a, w, y)
        torch.cuda.synchronize(dev)

    # sampling runs from just before the timed region (under the same load) to its end
    sampler = ClockSampler(torch.cuda.current_device()).start(keep_busy=busy)
    t_var = {}
    for gname, fn in variants.items():
        barrier()
        ev_step = timed(fn, args.steps)              # the timed region: exactly K steps
        barrier()
        t_v = sum(a_.elapsed_time(b_) * 1e-3 for a_, b_ in ev_step) / args.steps
        if sharded:                                  # max over ranks
            tt = torch.tensor([t_v], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_v = float(tt.item())
        t_var[gname] = t_v
    clocks = sampler.stop()
    gather_used = min(t_var, key=t_var.get)
    t_step = t_var[gather_used]
    step = variants[gather_used]
    # per-kernel split (same inputs, separate untimed-for-value loops) for the rooflines
    nk = min(args.steps, 50)
    ev_k1 = timed(lambda: act_quant_into(x, w.fmt, had, a.codes, a.sf, a.tensor_scale_dev, a.scratch), nk)
    ev_k2 = timed(lambda: P.gemm(a, w, y), nk)
    if fused_decode:   # the one kernel of the step (K1 and K2 above: the two-kernel path, for reference)
        ev_kd = timed(step_nccl, nk)
    torch.cuda.synchronize(dev)
    k1_mean = sum(a_.elapsed_time(b_) for a_, b_ in ev_k1) / nk * 1e-3
    k2_mean = sum(a_.elapsed_time(b_) for a_, b_ in ev_k2) / nk * 1e-3
    kd_mean = sum(a_.elapsed_time(b_) for a_, b_ in ev_kd) / nk * 1e-3 if fused_decode else None
    flops = 2.0 * M * N * K  # whole job (all ranks together compute the full N)
    value = flops / t_step / 1e12

    # ---------------- cuBLAS bf16 of the same layer (primary comparator)
    wb = w_dense if not sharded else w_dense[rank * w.N:(rank + 1) * w.N]
    yb = torch.empty((M, wb.shape[0]), dtype=torch.bfloat16, device=dev)
    for _ in range(args.warmup):
        torch.matmul(x, wb.t(), out=yb)
    tb = []
    nb = min(args.steps, 50)
    for _ in range(nb):
        flush_l2()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        torch.matmul(x, wb.t(), out=yb)
        e1.record(stream)
        tb.append((e0, e1))
    torch.cuda.synchronize(dev)
    t_bf16 = sum(e0.elapsed_time(e1) for e0, e1 in tb) / nb * 1e-3

    # ---------------- end to end through the public API, host buffers
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        yh = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
        xd = torch.empty_like(x)
        ne = min(args.steps, 20)

        def e2e_step():
            if sharded:
                xd.copy_(xh, non_blocking=True)
                yh.copy_(P.quantized_linear_sharded(xd, w), non_blocking=True)
            else:   # public host-buffer API: H2D, K1 + K2 and D2H pipelined over row chunks
                P.quantized_linear_host(xh, w, out=yh)

        for _ in range(3):
            e2e_step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ne):
            e2e_step()
        e1.record(stream)
        barrier()
        t_e2e = e0.elapsed_time(e1) * 1e-3 / ne
        if sharded:
            tt = torch.tensor([t_e2e], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        e2e = {"value": flops / t_e2e / 1e12, "unit": "TFLOP/s", "ms_per_step": t_e2e * 1e3,
               "h2d_bytes_per_step": xh.numel() * xh.element_size(),
               "d2h_bytes_per_step": yh.numel() * yh.element_size()}

    if rank != 0:
        if sharded:
            dist.destroy_process_group()
        return

    hbm, bf16_burst, bf16_sust, peak_src = peaks()
    G = 32 if fmt == "mxfp4" else 16
    k1_bytes = M * K * (2 + 0.5 + 1.0 / G) + (4 if fmt == "nvfp4" else 0)
    k2_flops = 2.0 * M * w.N * K
    fp4_peak = 4.0 * bf16_burst
    # K2's algorithmic bytes: A and W codes + scales once, bf16 output once.  Below the ridge
    # point (decode-sized M) K2 streams the weight and is HBM-bound; above it, tensor-bound.
    k2_bytes = (M + w.N) * K * (0.5 + 1.0 / G) + 2.0 * M * w.N
    k2_hbm_bound = k2_flops / k2_bytes < fp4_peak * 1e12 / (hbm * 1e9)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{args.config}:{'kd' if fused_decode else 'k2'}")
        except Exception:
            traffic = None

    # ---------------- sustained: the same step back to back for >= 4 s (SURVEY.md 8(d) "4 s
    # loop"; the headline above is the burst-clock figure), clocks sampled over the loop
    sustained = None
    if world == 1 and not args.no_sustained:
        samp = ClockSampler(torch.cuda.current_device()).start(keep_busy=busy)
        dev_s, n_s, t_wall = 0.0, 0, time.perf_counter()
        while time.perf_counter() - t_wall < 4.0:
            ev_s = timed(step, 100)
            torch.cuda.synchronize(dev)
            dev_s += sum(a_.elapsed_time(b_) * 1e-3 for a_, b_ in ev_s)
            n_s += len(ev_s)
        sustained = {"seconds": time.perf_counter() - t_wall, "steps": n_s, "ms_per_step": dev_s / n_s * 1e3,
                     "value": flops / (dev_s / n_s) / 1e12, "unit": "TFLOP/s", "clocks": samp.stop(),
                     "note": "L2 flushed between steps as in the timed region"}

    # ---------------- same-box FP4 comparators on THIS step's operands (
    # context, not parity oracles): cuBLASLt / flashinfer / vLLM-CUTLASS / QuTLASS GEMMs and the
    # QuTLASS rotate + quantize kernels
    comparators = None
    if world == 1 and not args.no_comparators:
        try:
            sys.path.insert(0, os.path.join(ROOT, "scripts"))
            import fp4_comparators
            act_quant_into(x, w.fmt, had, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
            with stdout_to_stderr():   # libraries print to fd 1; the bench prints ONE JSON line
                comparators = fp4_comparators.run(x, a, w, fmt, had, flush_l2)
            comparators["ours_k2"] = {"us": k2_mean * 1e6, "tflops": k2_flops / k2_mean / 1e12}
            comparators["ours_k1"] = {"us": k1_mean * 1e6, "gbs": k1_bytes / k1_mean / 1e9}
        except Exception as e:  # noqa: BLE001 - optional context
            comparators = {"error": f"{type(e).__name__}: {str(e)[:200]}"}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        arm = CpuArm(K, N, fmt, had)
        Ms = arm.rows_for(1.0, M)          # bounded sample: ~1 s per step, >= 8 s in all
        X = arm.inputs(Ms)
        arm.step(X)
        reps, t0 = 0, time.perf_counter()
        while reps < 3 or time.perf_counter() - t0 < 8.0:
            arm.step(X)
            reps += 1
        tc = (time.perf_counter() - t0) / reps
        cpu = {"value": 2.0 * Ms * N * K / tc / 1e12, "unit": "TFLOP/s", "cores": len(os.sched_getaffinity(0)),
               "kind": arm.kind, "blas": blas_threads(),
               "sample": f"{Ms} of {M} token rows, quantize_rtn + dequantize + float64 matmul, {reps} reps "
                         f"({'stock microfp from oracle/_ref' if arm.mf else 'numpy port'})"}

    if fused_decode:   # the step's one kernel: weight-stream bound (W codes + scales, X in, Y out)
        kd_bytes = k2_bytes + 2.0 * M * K + 4
        k2_roof = {"bound": "hbm", "kernel": "k_linear_decode (K1 + K2 in one launch)",
                   "achieved": kd_bytes / kd_mean / 1e9, "peak": hbm, "unit": "GB/s",
                   "frac": kd_bytes / kd_mean / 1e9 / hbm,
                   "note": f"{kd_bytes / 1e6:.2f} MB algorithmic (W codes and scales, bf16 X in, bf16 Y out) per launch",
                   "us": kd_mean * 1e6, "traffic": traffic}
    elif k2_hbm_bound:
        k2_roof = {"bound": "hbm", "kernel": "k_gemm_fp4 (K2)", "achieved": k2_bytes / k2_mean / 1e9,
                   "peak": hbm, "unit": "GB/s", "frac": k2_bytes / k2_mean / 1e9 / hbm,
                   "note": f"{k2_bytes / 1e6:.2f} MB algorithmic (A + W codes and scales, bf16 out) per launch",
                   "traffic": traffic}
    else:
        k2_roof = {"bound": "tensor", "kernel": "k_gemm_fp4 (K2)", "achieved": k2_flops / k2_mean / 1e12,
                   "peak": fp4_peak, "unit": "TFLOP/s", "frac": k2_flops / k2_mean / 1e12 / fp4_peak,
                   "peak_note": f"4x {peak_src} bf16 burst {bf16_burst} TF/s (PAPER.md:566 'out of 4x')",
                   "traffic": traffic}
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "fp4-e2m1 (fp32 accum)",
        "data": "synthetic: bf16 N(0,1) activations, N(0,1/K) random-init weights (GPU RTN)",
        # config: the workload only, key for key the reference arm's (run details below)
        "config": {"workload": name, "M": M, "K": K, "N": N, "format": fmt, "hadamard": had},
        "parallelism": f"N-shard x{world}" if sharded else "single",
        "gather": gather_used if sharded else None,
        "l2": "flushed between steps (256 MiB memset + 256 MiB read sweep)",
        "k1_us": k1_mean * 1e6, "k2_us": k2_mean * 1e6,
        "gather_ms_per_step": {k_: v_ * 1e3 for k_, v_ in t_var.items()} if sharded else None,
        "gemm_tflops_per_gpu": k2_flops / k2_mean / 1e12,
        "rotquant_gbs": k1_bytes / k1_mean / 1e9,
        "bf16_cublas_us": t_bf16 * 1e6, "bf16_cublas_tflops": 2.0 * M * wb.shape[0] * K / t_bf16 / 1e12,
        "speedup_vs_cublas_bf16": t_bf16 / t_step,
        "roofline": k2_roof,
        "roofline_k1": {"bound": "hbm", "kernel": "k_act_quant (K1)", "achieved": k1_bytes / k1_mean / 1e9,
                        "peak": hbm, "unit": "GB/s", "frac": k1_bytes / k1_mean / 1e9 / hbm},
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "sustained": sustained, "comparators": comparators,
        "gpu_launches": launches_per_step * args.steps,
    }
    print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
