"""Randomised fast-path parity sweep at sizes the unit tests do not reach:
    python tools/stress_parity.py [seed0] [n_seeds] [options_per_seed]
Each seed draws a mixed batch (European / American call / BSM put) over the
broad ranges of tests/test_gpu_random.py but with T up to 131 072, most of
them not powers of two (the goldens and bench configs are), prices it in ONE
device batch (fast method) and checks every option against the oracle port
(oracle/port.py, a fork pool over the host cores): status class, price within
1e-9 max(|ref|, K), boundary records equal except at oracle-certified ties.
Prints one line per seed and a summary; exit code 1 on any mismatch.
Tool only: the product never imports oracle/."""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import NMARG, boundary_check, price_close  # noqa: E402
from oracle import port  # noqa: E402

NAMES = {0: "euro", 1: "call", 2: "put"}
T_SET = [2, 5, 129, 255, 511, 777, 1025, 2047, 4097, 5000, 8191, 10007, 12345, 16385, 20011, 30000, 32767,
         40009, 50000, 65535, 65537, 70001, 99991, 100000, 131071, 131072]
ERRS = {0x100: "ValidationError", 0x200: "StabilityError", 0x300: "DomainError", 0x400: "GeometryError",
        0x500: "NumericalIntegrityError", 0x600: "ValueError"}


def draw(rng, n):
    rows = []
    while len(rows) < n:
        kind = int(rng.integers(0, 3))
        S = float(np.exp(rng.uniform(np.log(5.0), np.log(500.0))))
        K = float(S * np.exp(rng.uniform(-1.0, 1.0)))
        R = float(rng.choice([0.0, 1e-4, rng.uniform(0.0, 0.15)]))
        Y = 0.0 if kind == 2 else float(rng.choice([0.0, 1e-4, rng.uniform(0.0, 0.12)]))
        V = float(rng.uniform(0.03, 1.0))
        E = float(rng.uniform(5.0, 1500.0))
        T = int(rng.choice(T_SET))
        rows.append((kind, S, K, R, Y, V, E, T))
    return rows


def oracle(row):
    kind, args = row[0], row[1:]
    k = NAMES[kind]
    try:
        if k == "euro":
            return "", port.euro_fast(*args), None
        p, t, c, m = port.call_fast(*args, margins=True) if k == "call" else port.put_fast(*args, margins=True)
        return "", p, (t, c, m)
    except port.OracleError as e:
        return e.kind, None, None
    except ValueError:
        return "ValueError", None, None


def main():
    seed0 = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    nseeds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 96
    from paper_2303_02317_b200 import _native

    pool = mp.get_context("fork").Pool(os.cpu_count())
    bad_total = 0
    checked = ties_total = errs_total = 0
    for seed in range(seed0, seed0 + nseeds):
        rng = np.random.default_rng([777, seed])
        rows = draw(rng, n)
        kind = np.array([r[0] for r in rows], dtype=np.int8)
        cols = [np.array([r[i] for r in rows]) for i in range(1, 7)]
        T = np.array([r[7] for r in rows], dtype=np.int64)
        t0 = time.time()
        res = _native.price_batch_full(kind, *cols, T, method=0, bnd_cap=64)
        t1 = time.time()
        ref = pool.map(oracle, rows, chunksize=1)
        t2 = time.time()
        bad = []
        for i, r in enumerate(rows):
            ek, p, bnd = ref[i]
            st = int(res.status[i])
            if ek:
                errs_total += 1
                if ERRS.get(st & 0xFF00) != ek:
                    bad.append((i, r, "status", ek, hex(st)))
                continue
            if st != 0:
                bad.append((i, r, "status", "ok", hex(st)))
                continue
            if not price_close(res.price[i], p, r[2]):
                bad.append((i, r, "price", res.price[i], p))
                continue
            degenerate = r[0] == 1 and r[3] <= 1e-4 and r[4] <= 1e-4
            if bnd is not None and not degenerate:
                t, c = res.boundary(i)
                ok, nt, why = boundary_check(r[0], r[2], t, c, bnd[0], bnd[1], bnd[2])
                ties_total += nt
                if not ok:
                    bad.append((i, r, "boundary", why))
        checked += len(rows)
        bad_total += len(bad)
        print(f"seed {seed}: {len(rows)} options, gpu {t1 - t0:.2f} s, oracle {t2 - t1:.1f} s, mismatches {len(bad)}",
              flush=True)
        for b in bad[:10]:
            print("   ", b, flush=True)
    print(f"checked {checked} options ({errs_total} reference errors matched by class, {ties_total} certified ties): "
          f"{bad_total} mismatches")
    sys.exit(1 if bad_total else 0)


if __name__ == "__main__":
    main()
