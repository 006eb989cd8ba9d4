"""O(T^2) baseline sweeps (north_star subsystem 3): one option
alone and a batch, register-resident sweep (fl_sweep.cu) vs the round-1
global-memory march (FL_NO_SWEEP=1), CUDA-event timing of fl_batch_run.

    python tools/sweep_bench.py            # prints one JSON line per case
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_cases():
    import torch

    from paper_2303_02317_b200 import _native

    torch.cuda.set_device(0)
    st = torch.cuda.current_stream().cuda_stream
    rows = []
    cases = [("put", 2, 4096, 1), ("call", 1, 4096, 1), ("euro", 0, 4096, 1), ("put", 2, 4096, 148),
             ("put", 2, 2048, 1), ("put", 2, 5000, 1), ("call", 1, 10000, 1)]
    for name, kind, T, n in cases:
        rng = np.random.default_rng(T + n)
        S = np.full(n, 100.0) if kind == 2 else rng.uniform(80, 120, n)  # put: spot on the strike node
        K = np.full(n, 100.0)
        R = np.full(n, 0.05)
        Y = np.full(n, 0.0 if kind == 2 else 0.03)
        V = rng.uniform(0.2, 0.4, n)
        E = np.full(n, 365.0)
        db = _native.DeviceBatch(np.full(n, kind, np.int8), S, K, R, Y, V, E, np.full(n, T, np.int64),
                                 method=_native.METHOD_BASELINE, bnd_cap=T + 2, stream=st)
        db.run(st)
        torch.cuda.synchronize()
        ms = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            db.run(st)
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        res = db.fetch(st)
        assert np.all(res.status == 0), (name, T, n, [hex(x) for x in res.status[:4]])
        cells = n * (T * T if kind == 2 else T * (T + 1) / 2)  # put: sum_s (2T+1-2s) ~ T^2
        t = float(np.median(ms))
        rows.append({"case": f"{name} T={T} x{n}", "ms": t, "cells_per_s": cells / (t * 1e-3),
                     "price0": float(res.price[0]), "sweep": os.environ.get("FL_NO_SWEEP") != "1"})
        db.close()
    return rows


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        print(json.dumps(run_cases()))
        sys.exit(0)
    out = {}
    for mode in ("sweep", "global"):
        env = dict(os.environ, FL_NO_SWEEP="1" if mode == "global" else "0")
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        if r.returncode:
            sys.exit(f"{mode} child failed:\n{r.stdout}\n{r.stderr}")
        out[mode] = json.loads(r.stdout.strip().splitlines()[-1])
    for a, b in zip(out["sweep"], out["global"]):
        assert a["price0"] == b["price0"] or abs(a["price0"] - b["price0"]) <= 1e-12 * abs(b["price0"]), (a, b)
        print(json.dumps({"case": a["case"], "sweep_ms": a["ms"], "global_ms": b["ms"],
                          "speedup": b["ms"] / a["ms"], "sweep_cells_per_s": a["cells_per_s"],
                          "bit_identical_price": a["price0"] == b["price0"]}))
