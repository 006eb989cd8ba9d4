"""Bench CSV on the GPU path.

Mirrors the reference's ``bench`` command (cli.py:619-720): same method names,
step lists, spec flags, median-of-reps wall time per (method, T), and the same
CSV schema ``method,T,seconds,price,reps`` -- so GPU timings sit beside the
reference's own bench output.  Every call goes through this package's
drop-in pricers (the device path).

    python -m paper_2303_02317_b200.benchcsv --method fast_put,fast_american --steps 4096,65536
"""

from __future__ import annotations

import argparse
import csv
import statistics
import sys
import time

from .american import fast_american_call
from .binomial import (
    baseline_american_call,
    baseline_european,
    closed_form_european,
    fast_european,
    gaussian_approx_european,
)
from .bsm import DEFAULT_LAMBDA, baseline_put_fd, fast_put_bsm
from .model import OptionSpec, UnsupportedCombinationError, ValidationError

__all__ = ["BENCH_METHODS", "bench_records", "main"]

BENCH_METHODS = ("fast_european", "baseline_european", "gaussian_european", "closed_form_european",
                 "fast_american", "baseline_american", "fast_put", "baseline_put")  # cli.py:623-632


def _call(method: str, spec: OptionSpec, lam: float) -> float:
    """cli.py:635-650."""
    if method == "fast_european":
        return fast_european(spec)
    if method == "baseline_european":
        return baseline_european(spec)
    if method == "gaussian_european":
        return gaussian_approx_european(spec)
    if method == "closed_form_european":
        return closed_form_european(spec)
    if method == "fast_american":
        return fast_american_call(spec).price
    if method == "baseline_american":
        return baseline_american_call(spec).price
    if method == "fast_put":
        return fast_put_bsm(spec, lam).price
    return baseline_put_fd(spec, lam).price


def bench_records(methods, steps: str, reps: int, spec: OptionSpec, lam: float = DEFAULT_LAMBDA):
    """(method, T, seconds, price, reps) rows as cmd_bench computes them."""
    for m in methods:
        if m not in BENCH_METHODS:
            raise UnsupportedCombinationError(f"unknown bench method {m!r}; choose from {', '.join(BENCH_METHODS)}")
    try:
        step_list = sorted({int(tok) for tok in steps.split(",") if tok})
    except ValueError as exc:
        raise ValidationError("steps", f"bad step list: {exc}") from None
    if not step_list or step_list[0] < 1:
        raise ValidationError("steps", "step counts must be positive")
    if reps < 1:
        raise ValidationError("reps", "reps must be >= 1")
    rows = []
    for m in methods:
        base = OptionSpec(spec.spot, spec.strike, spec.rate, spec.dividend_yield, spec.volatility,
                          spec.days_to_expiry, step_list[0])
        _call(m, base, lam)  # warm-up (library load, twiddles, workspaces)
        for T in step_list:
            s = OptionSpec(base.spot, base.strike, base.rate, base.dividend_yield, base.volatility,
                           base.days_to_expiry, T)
            price, timings = 0.0, []
            for _ in range(reps):
                t0 = time.perf_counter()
                price = float(_call(m, s, lam))
                timings.append(time.perf_counter() - t0)
            rows.append((m, T, statistics.median(timings), price, reps))
    return rows


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="time the GPU pricers (fftlattice bench CSV schema)")
    ap.add_argument("--method", required=True)
    ap.add_argument("--steps", required=True)
    ap.add_argument("--spot", type=float, default=100.0)
    ap.add_argument("--strike", type=float, default=100.0)
    ap.add_argument("--rate", type=float, default=0.05)
    ap.add_argument("--yield", dest="dividend_yield", type=float, default=0.03)
    ap.add_argument("--vol", type=float, default=0.2)
    ap.add_argument("--days", type=int, default=365)
    ap.add_argument("--lambda", dest="lam", type=float, default=DEFAULT_LAMBDA)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--csv", default=None)
    ap.add_argument("--parallel", action="store_true", help="accepted for compatibility (no effect)")
    a = ap.parse_args(argv)
    methods = [m.strip() for m in a.method.split(",") if m.strip()]
    spec = OptionSpec(a.spot, a.strike, a.rate, a.dividend_yield, a.vol, a.days, 1)
    rows = bench_records(methods, a.steps, a.reps, spec, a.lam)
    out = open(a.csv, "w", newline="") if a.csv else sys.stdout
    try:
        w = csv.writer(out)
        w.writerow(["method", "T", "seconds", "price", "reps"])
        for m, T, sec, price, reps in rows:
            w.writerow([m, str(T), repr(sec), repr(price), str(reps)])
    finally:
        if out is not sys.stdout:
            out.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
