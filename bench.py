#!/usr/bin/env python
"""Benchmark of the B200-native fftlattice pricing path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload put16|c1|c2|c3|c4|c5] [--batch B]

Metric (BASELINE.json): options priced per second, fp64.  Default workload =
the headline: BSM American puts at T=2^16 drawn from the C3
distribution, batch 256 per GPU (weak scaling: rank r prices its own seeded
shard; the batch-1024 figure rides along in ``also``).  A step is one pass of
the hot path over the batch:

* ``value``: device-resident inputs (fl_batch_prepare once), step = one
  fl_batch_run (for put16 exactly one launch of the persistent put kernel);
  CUDA events on the launch stream; L2 flushed between timed steps (256 MiB
  write, outside the events); max over ranks.
* ``e2e``: the reference-facing C-ABI call ``fl_price_batch`` with host numpy
  buffers, every step: host parameter derivation, pinned H2D of the
  per-option records, kernels, D2H of prices / status.
* ``roofline``: the FP64 pipe (the path is fp64 FFT + explicit stencil work,
  not a tensor-core contraction).  achieved = REFERENCE-ALGORITHMIC flops of
  the batch (counted live by the kernel as it walks the reference's own
  decomposition: 5 flops per projected cell of each reference strip,
  5 N log2 N + 6 (N/2+1) per reference FFT jump) / the kernel's
  mean duration; peak = DFMA throughput probed live on this GPU
  (MEASURED_PEAKS.json carries no fp64 figure); traffic = DRAM bytes per
  launch from the committed ncu capture (profiles/ncu_traffic.json) or null.
* ``cpu_baseline``: the oracle port (numpy pocketfft + C loops restating the
  reference) on a bounded sample of the same workload, all host cores.

``--impl reference`` times that CPU reference on the same config instead
(rank 0 only; the reference is pure Python, so its CPU path is the oracle).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2303_02317_b200.shard import lpt_shards  # noqa: E402
from paper_2303_02317_b200.workloads import draw_config  # noqa: E402

METRIC = "options priced/sec (fp64, T=2^16) and achieved fraction of FP64/HBM roofline"

WORKLOADS = {
    "put16": dict(config=6, desc="BSM American put (lambda 0.4), C3 ranges, T=2^16, 256 options per GPU"),
    "c1": dict(config=1, desc="C1 binomial European call, 1024 options, T=4096"),
    "c2": dict(config=2, desc="C2 binomial American call, 256 options, T=2^14"),
    "c3": dict(config=3, desc="C3 BSM American put, 256 options, T=2^14"),
    "c4": dict(config=4, desc="C4 64 puts + 64 American calls, T=2^18"),
    "c5": dict(config=5, desc="C5 mixed 65536 options, T=2^U{10..16}, LPT-sharded"),
}


def rank_info():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def make_batch(args, rank, world):
    """(local batch, global option count, scaling, local indices)."""
    wl = WORKLOADS[args.workload]
    if args.workload == "put16":
        per = args.batch or 256
        full = draw_config(6, n=per * world)
        idx = np.arange(rank * per, (rank + 1) * per)
        return full.subset(idx), per * world, "weak", idx
    full = draw_config(wl["config"], n=args.batch or None)
    idx = lpt_shards(full.kind, full.T, world)[rank] if world > 1 else np.arange(len(full))
    return full.subset(idx), len(full), "strong", idx


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


# ---------------------------------------------------------------------------
# CPU reference (oracle port) -- only this leg and the reference arm touch oracle/


def cpu_reference(batch, max_options: int | None = None):
    """Oracle port (restatement of the reference, pinned to its goldens) on all host cores."""
    import multiprocessing as mp

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cores = os.cpu_count() or 1
    n = len(batch)
    take = min(n, max_options if max_options else n)
    items = [(int(batch.kind[i]),) + tuple(float(getattr(batch, f)[i]) for f in "SKRYVE") + (int(batch.T[i]),)
             for i in range(take)]
    ctx = mp.get_context("fork")
    with ctx.Pool(processes=cores, initializer=_pool_init) as pool:
        pool.map(_price_one, items[:1] * cores)  # warm-up: load the C loops in every worker
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
    batch, total, scaling, _ = make_batch(args, 0, 1)
    wl = WORKLOADS[args.workload]
    cores = os.cpu_count() or 1
    per_step = max(cores, 8)
    vals = []
    for s in range(args.warmup + args.steps):
        lo = (s * per_step) % len(batch)
        sub = batch.subset(np.arange(lo, lo + per_step) % len(batch))
        take, wall, cores_used, _ = cpu_reference(sub)
        if s >= args.warmup:
            vals.append((take, wall))
    opts = sum(t for t, _ in vals)
    secs = sum(w for _, w in vals)
    v = opts / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "options/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / len(vals),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE ranges)",
        "config": {"workload": wl["desc"], "options_per_step": per_step},
        "cpu_baseline": {"value": v, "unit": "options/s", "cores": cores_used, "kind": "port",
                         "sample": f"{per_step} options per step from the {args.workload} workload; oracle/port.py "
                                   "(the reference's algorithm restated: numpy pocketfft + C loops), "
                                   f"{cores_used} worker processes"},
        "e2e": {"value": v, "unit": "options/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------


def ncu_traffic(workload: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except (OSError, ValueError):
        return None


def time_steps(db, sh, stream, steps, flush):
    import torch

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s in range(steps):
        flush.zero_()
        ev[s][0].record(stream)
        db.run(sh)
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="put16")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the batch-1024 side measurement")
    ap.add_argument("--cpu-sample", type=int, default=32, help="options in the cpu_baseline sample")
    args = ap.parse_args()
    rank, world, local = rank_info()
    args.warmup = max(args.warmup, 3)

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
    batch, total, scaling, local_idx = make_batch(args, rank, world)

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

    clk = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    time.sleep(0.3)
    step_ms = time_steps(db, sh, stream, args.steps, flush)
    clocks = clk.stop()
    t_ms = sum(step_ms)
    if dist:
        tt = torch.tensor([t_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
        dist.barrier()
    value = total * args.steps / (t_ms / 1e3)

    # e2e: the reference-facing call with host buffers, every step
    e2e_ms = []
    for s in range(args.steps + 1):
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
        from paper_2303_02317_b200.shard import gather_prices

        gather_prices(local_idx, r.price, r.status, total, dist, rank)  # results land on rank 0 (untimed)
    n_local = len(batch)

    # batch-1024 side figure for the headline, single GPU only
    also = {}
    if args.workload == "put16" and world == 1 and not args.no_extra:
        b4 = draw_config(6, n=1024)
        db4 = _native.DeviceBatch(b4.kind, b4.S, b4.K, b4.R, b4.Y, b4.V, b4.E, b4.T, lam=0.4, stream=sh)
        for _ in range(2):
            db4.run(sh)
        ms4 = time_steps(db4, sh, stream, 2, flush)
        st4 = db4.stats(sh)
        k4 = sum(ms4) / len(ms4)
        also["batch_1024"] = {"value": 1024 / (k4 / 1e3), "unit": "options/s", "ms_per_step": k4,
                              "roofline_frac": (st4["ref_flops"] / (k4 * 1e-3) / 1e12) / peak if peak else None}
        db4.close()

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    mean_ms = t_ms / args.steps
    achieved = stats["ref_flops"] / (mean_ms * 1e-3) / 1e12
    line = {
        "metric": METRIC,
        "value": value, "unit": "options/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": mean_ms, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded draws, BASELINE.json ranges)",
        "config": {"workload": WORKLOADS[args.workload]["desc"], "options_per_step": total,
                   "options_per_gpu": n_local, "lambda": 0.4, "put_cutoff": 128, "call_cutoff": 256,
                   "l2": "flushed between timed steps (256 MiB write outside the events); the chain "
                         "arenas (~3 MB per option) exceed L2 as well",
                   "parallelism": f"option-sharded x{world}, no collective on the data path",
                   "device_bytes_per_gpu": db.device_bytes()},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None,
                     "traffic": ncu_traffic(args.workload),
                     "peak_source": "measured live: fl_probe_fp64 DFMA throughput on this GPU "
                                    "(MEASURED_PEAKS.json has no fp64 entry)",
                     "kernel": {"put16": "put_fast_kernel", "c3": "put_fast_kernel", "c2": "call_fast_kernel",
                                "c1": "euro_fast_kernel"}.get(args.workload, "all fast kernels of the step"),
                     "ref_algorithmic_flops_per_step": stats["ref_flops"],
                     "executed_flops_per_step": stats["fp64_flops"]},
        "e2e": {"value": (total if scaling == "strong" else n_local * world) / (e2e_t / 1e3),
                "unit": "options/s", "ms_per_step": e2e_t,
                "h2d_bytes_per_step": stats["h2d_bytes"], "d2h_bytes_per_step": 16 * n_local},
        "clocks": clocks,
        "gpu_launches": launches_per_step * args.steps,
        "status_errors": bad,
    }
    if also:
        line["also"] = also
    if not args.no_cpu_baseline and world == 1:
        sample = min(args.cpu_sample, n_local)
        take, wall, cores, cpu_prices = cpu_reference(batch, sample)
        cpu_prices = np.asarray(cpu_prices)
        rel = np.abs(res.price[:take] - cpu_prices) / np.maximum(np.abs(cpu_prices), batch.K[:take])
        line["cpu_baseline"] = {
            "value": take / wall, "unit": "options/s", "cores": cores, "kind": "port",
            "sample": f"first {take} options of this workload, oracle/port.py (the reference's algorithm "
                      f"restated, pinned to its goldens), {cores} worker processes"}
        line["parity_vs_cpu"] = {"options": int(take), "max_abs_err_over_max_ref_K": float(np.nanmax(rel))}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
