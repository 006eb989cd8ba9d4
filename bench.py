#!/usr/bin/env python
"""Benchmark of the B200-native fftlattice pricing path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload put16|c1|c2|c3|c4|c5] [--batch B]

Metric (BASELINE.json): options priced per second, fp64.  Default workload =
the headline: BSM American puts at T=2^16 drawn from the C3 distribution,
batch 256 per GPU (weak scaling: rank r prices its own seeded shard).  A step
is one pass of the hot path over the batch:

* ``value``: device-resident inputs (fl_batch_prepare once), step = one
  fl_batch_run (the persistent put D&C kernel); CUDA events on the launch
  stream; L2 flushed between timed steps (256 MiB write) outside the events.
* ``e2e``: the reference-facing call ``fl_price_batch`` with host buffers:
  host parameter derivation, pinned H2D of the per-option records, kernels,
  D2H of prices/status, every step.
* ``roofline``: FP64 pipe (the path is fp64 FFT + explicit stencil work, not a
  tensor-core contraction).  achieved = fp64 flops the kernel executed (counted
  on device: 5 C log2 C per complex FFT, 5 per explicit cell) / kernel time;
  peak = DFMA throughput probed live on this GPU (fl_probe_fp64).
* ``cpu_baseline``: the oracle port (numpy pocketfft + C loops, bit-exact with
  the reference) on a bounded sample of the same workload, all host cores.

``--impl reference`` times that CPU reference on the same config instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2303_02317_b200.workloads import KIND_PUT, draw_config  # noqa: E402

WORKLOADS = {
    "put16": dict(config=6, T=2 ** 16, desc="BSM American put (lambda 0.4), C3 ranges, T=2^16"),
    "c1": dict(config=1, T=4096, desc="C1 binomial European call, T=4096"),
    "c2": dict(config=2, T=2 ** 14, desc="C2 binomial American call, T=2^14"),
    "c3": dict(config=3, T=2 ** 14, desc="C3 BSM American put, T=2^14"),
    "c4": dict(config=4, T=2 ** 18, desc="C4 64 puts + 64 American calls, T=2^18"),
    "c5": dict(config=5, T=None, desc="C5 mixed 65536 options, T=2^U{10..16}, LPT-sharded"),
}


def rank_info():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def lpt_shards(batch, nshard):
    """Cost-balanced longest-processing-time partition."""
    T = batch.T.astype(np.float64)
    l2 = np.log2(np.maximum(T, 2.0))
    c = np.where(batch.kind == 2, 24.8, np.where(batch.kind == 1, 10.0, 0.05)) * T * np.maximum(l2, 1) ** 2
    order = np.argsort(-c, kind="stable")
    load = np.zeros(nshard)
    owner = np.empty(len(c), dtype=np.int64)
    for i in order:
        r = int(np.argmin(load))
        owner[i] = r
        load[r] += c[i]
    return [np.nonzero(owner == r)[0] for r in range(nshard)]


def make_batch(args, rank, world):
    wl = WORKLOADS[args.workload]
    if args.workload == "c5":
        full = draw_config(5, n=args.batch if args.batch else None)
        idx = lpt_shards(full, world)[rank]
        return full.subset(idx), len(full), "strong"
    if args.workload in ("c1", "c2", "c3", "c4"):
        full = draw_config(wl["config"])
        if world > 1:
            shards = np.array_split(np.arange(len(full)), world)
            return full.subset(shards[rank]), len(full), "strong"
        return full, len(full), "strong"
    per = args.batch or 256
    full = draw_config(6, n=per * world)
    return full.subset(np.arange(rank * per, (rank + 1) * per)), per * world, "weak"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.gpu = gpu_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference(batch, wall_budget_s: float, max_options: int | None = None):
    """Oracle port (bit-exact restatement of the reference) on all host cores."""
    import multiprocessing as mp

    from oracle import port  # only the cpu_baseline / reference arm may import the oracle

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cores = os.cpu_count() or 1
    n = len(batch)
    take = min(n, max_options if max_options else n)
    items = [(int(batch.kind[i]),) + tuple(float(getattr(batch, f)[i]) for f in "SKRYVE") + (int(batch.T[i]),)
             for i in range(take)]
    ctx = mp.get_context("fork")
    with ctx.Pool(processes=cores, initializer=_pool_init) as pool:
        pool.map(_price_one, items[:cores])  # warm-up (numba-free; builds/loads the C loops)
        t0 = time.perf_counter()
        prices = pool.map(_price_one, items, chunksize=1)
        wall = time.perf_counter() - t0
    return take, wall, cores, prices


def _pool_init():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"


def _price_one(item):
    from oracle import port

    kind, S, K, R, Y, V, E, T = item
    name = {0: "euro", 1: "call", 2: "put"}[kind]
    try:
        return port.price(name, S, K, R, Y, V, E, T)
    except port.OracleError:
        return float("nan")


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    batch, total, scaling = make_batch(args, 0, 1)
    wl = WORKLOADS[args.workload]
    cores = os.cpu_count() or 1
    per_step = max(cores, 16)
    vals = []
    for s in range(args.warmup + args.steps):
        sub = batch.subset(np.arange((s * per_step) % len(batch), (s * per_step) % len(batch) + per_step)
                           % len(batch))
        take, wall, cores_used, _ = cpu_reference(sub, 60.0)
        if s >= args.warmup:
            vals.append((take, wall))
    opts = sum(t for t, _ in vals)
    secs = sum(w for _, w in vals)
    v = opts / secs
    line = {
        "impl": "reference", "metric": "options priced/sec (fp64)", "value": v, "unit": "options/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / len(vals),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE ranges)",
        "config": {"workload": wl["desc"], "batch_per_step": per_step},
        "cpu_baseline": {"value": v, "unit": "options/s", "cores": cores_used, "kind": "port",
                         "sample": f"{per_step} options per step of the {args.workload} workload; oracle/port.py "
                                   "(bit-exact restatement of the reference: numpy pocketfft + C loops)"},
        "e2e": {"value": v, "unit": "options/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="put16")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=32, help="options in the cpu_baseline sample")
    args = ap.parse_args()
    rank, world, local = rank_info()

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2303_02317_b200 import _native

    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    batch, total, scaling = make_batch(args, rank, world)
    args.warmup = max(args.warmup, 3)

    peak = _native.probe_fp64_tflops(sh)
    db = _native.DeviceBatch(batch.kind, batch.S, batch.K, batch.R, batch.Y, batch.V, batch.E, batch.T,
                             lam=0.4, stream=sh)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        db.run(sh)
    torch.cuda.synchronize()
    res = db.fetch(sh)
    stats = db.stats(sh)
    launches_per_step = db.launches()
    bad = int(np.sum(res.status != 0))

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clk = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    time.sleep(0.3)
    for s in range(args.steps):
        flush.zero_()
        ev[s][0].record(stream)
        db.run(sh)
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_ms = sum(step_ms)
    if dist:
        tt = torch.tensor([t_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
        dist.barrier()
    value = total * args.steps / (t_ms / 1e3)

    # e2e: the reference-facing call with host buffers, every step
    e2e_ms = []
    for s in range(max(2, min(args.steps, 5))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r = _native.price_batch(batch.kind, batch.S, batch.K, batch.R, batch.Y, batch.V, batch.E, batch.T,
                                lam=0.4, stream=sh)
        b.record(stream)
        torch.cuda.synchronize()
        if s > 0:
            e2e_ms.append(a.elapsed_time(b))
    e2e_t = sum(e2e_ms) / len(e2e_ms)
    if dist:
        tt = torch.tensor([e2e_t], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())
    n_local = len(batch)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    mean_ms = t_ms / args.steps
    flops = stats["fp64_flops"]
    achieved = flops / (mean_ms * 1e-3) / 1e12
    ref_flops = None
    if args.workload in ("put16", "c3"):
        T = float(WORKLOADS[args.workload]["T"])
        ref_flops = 24.8 * T * math.log2(T) ** 2 * n_local
    line = {
        "metric": "options priced/sec (fp64, T=2^16) and achieved fraction of FP64/HBM roofline",
        "value": value, "unit": "options/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded draws, BASELINE.json ranges)",
        "config": {"workload": WORKLOADS[args.workload]["desc"], "options_per_step": total,
                   "options_per_gpu": n_local, "lambda": 0.4, "put_cutoff": 128, "call_cutoff": 256,
                   "l2": "flushed between timed steps (256 MiB write outside the events)",
                   "parallelism": f"option-sharded x{world}, no collective on the data path"},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None, "traffic": None,
                     "peak_source": "measured live: fl_probe_fp64 DFMA throughput on this GPU",
                     "kernel": "put_fast_kernel" if args.workload in ("put16", "c3") else "mixed",
                     "flops_per_step": flops,
                     "ref_equiv_tflops": (ref_flops / (mean_ms * 1e-3) / 1e12) if ref_flops else None},
        "e2e": {"value": total / (e2e_t / 1e3) if scaling == "strong" else n_local * world / (e2e_t / 1e3),
                "unit": "options/s", "ms_per_step": e2e_t,
                "h2d_bytes_per_step": stats["h2d_bytes"], "d2h_bytes_per_step": 16 * n_local},
        "clocks": clocks,
        "gpu_launches": launches_per_step * args.steps,
        "status_errors": bad,
    }
    if not args.no_cpu_baseline and world == 1:
        sample = min(args.cpu_sample, n_local)
        take, wall, cores, cpu_prices = cpu_reference(batch, 30.0, sample)
        cpu_prices = np.asarray(cpu_prices)
        rel = np.abs(res.price[:take] - cpu_prices) / np.maximum(np.abs(cpu_prices), batch.K[:take])
        line["cpu_baseline"] = {
            "value": take / wall, "unit": "options/s", "cores": cores, "kind": "port",
            "sample": f"first {take} options of this workload, oracle/port.py (bit-exact reference restatement), "
                      f"{cores} worker processes"}
        line["parity_vs_cpu"] = {"options": int(take), "max_abs_err_over_max_ref_K": float(np.nanmax(rel))}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
