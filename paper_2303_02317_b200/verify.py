"""Randomised oracle and invariant suites on the GPU path.

Mirrors the reference's ``verify`` command (cli.py:208-616: the same six
suites, the same seeded draws ``default_rng([seed, suite_index])``, the same
tolerances, output lines and exit code), with every price, boundary and grid
computed by the device: each suite draws its specs first and prices them in
batched device calls (fast and O(T^2) baselines), the boundary-lemma suite
checks cell-exact lemmas on full device grids (``keep_grid``).

    python -m paper_2303_02317_b200.verify [--steps 1024] [--seed 0] [--reps 25]
"""

from __future__ import annotations

import argparse
import math
import sys

import numpy as np

from . import _native
from .american import fast_american_call
from .binomial import baseline_american_call, baseline_european
from .bsm import baseline_put_fd, bsm_green_value, discretize_bsm, fast_put_bsm
from .fft import Kernel, apply_linear_steps, convolve, fft_forward, fft_inverse, kernel_power
from .model import NO_GREEN, DomainError, GridRow, OptionSpec, StabilityError, ValidationError, derive_binomial_params

__all__ = ["check_boundary_lemmas", "run_suites", "main"]


def _draw_spec(rng, *, moneyness_band=None) -> OptionSpec:
    """cli.py:208-243 (same draw order)."""
    while True:
        spot = float(rng.uniform(50.0, 200.0))
        strike = float(rng.uniform(50.0, 200.0))
        rate = float(rng.uniform(0.01, 0.1))
        dividend_yield = float(rng.uniform(0.01, 0.1))
        vol = float(rng.uniform(0.1, 0.5))
        days = int(rng.integers(30, 731))
        if moneyness_band is not None:
            years = days / 365.0
            drift = (rate - dividend_yield - 0.5 * vol * vol) * years
            score = (math.log(spot / strike) + drift) / (vol * math.sqrt(years))
            if not -moneyness_band <= score <= moneyness_band:
                continue
        return OptionSpec(spot, strike, rate, dividend_yield, vol, days, 1)


def _with_steps(spec: OptionSpec, steps: int) -> OptionSpec:
    return OptionSpec(spec.spot, spec.strike, spec.rate, spec.dividend_yield, spec.volatility,
                      spec.days_to_expiry, steps)


def _rel_err(value, oracle, scale):
    return abs(value - oracle) / max(abs(oracle), 1e-9 * scale)


def _spec_line(s: OptionSpec) -> str:
    return (f"spot={s.spot!r} strike={s.strike!r} rate={s.rate!r} yield={s.dividend_yield!r} "
            f"vol={s.volatility!r} days={s.days_to_expiry} steps={s.steps}")


def _batch(kind, specs, method, **kw):
    """Price specs of one kind in one device call: (price, status, BatchResult)."""
    cols = [np.array([getattr(s, f) for s in specs], dtype=np.float64)
            for f in ("spot", "strike", "rate", "dividend_yield", "volatility", "days_to_expiry")]
    T = np.array([s.steps for s in specs], dtype=np.int64)
    cap = int(T.max()) + 2 if method == _native.METHOD_BASELINE else 64
    res = _native.price_batch_full(np.int8(kind), *cols, T, method=method, bnd_cap=cap, **kw)
    for i, st in enumerate(res.status):
        err = _native.status_error(int(st))
        if err is not None:
            raise err
    return res


def _suite_fft(rng, trials, max_steps):
    """cli.py:271-346 on the device transforms / correlations."""
    worst, failures = 0.0, []
    for _ in range(trials):
        size = 2 ** int(rng.integers(0, 10))
        vec = rng.standard_normal(size) + 1j * rng.standard_normal(size)
        err = float(np.max(np.abs(fft_inverse(fft_forward(vec)) - vec))) / 1e-12
        worst = max(worst, err)
        if err > 1.0:
            failures.append(f"round-trip size={size} err-ratio={err:.3g}")
        a = rng.standard_normal(int(rng.integers(1, 65)))
        b = rng.standard_normal(int(rng.integers(1, 65)))
        got, ref = convolve(a, b), np.convolve(a, b)
        err = float(np.max(np.abs(got - ref))) / max(1.0, float(np.max(np.abs(ref)))) / 1e-10
        worst = max(worst, err)
        if err > 1.0:
            failures.append(f"convolve sizes=({len(a)},{len(b)}) err-ratio={err:.3g}")
        nw = int(rng.integers(2, 4))
        weights = rng.uniform(0.1, 0.9, size=nw)
        weights /= weights.sum()
        power = int(rng.integers(0, 7))
        kern = Kernel(weights=weights, min_offset=int(rng.integers(-2, 3)))
        got_k = kernel_power(kern, power)
        ref_w = np.array([1.0])
        for _ in range(power):
            ref_w = np.convolve(ref_w, weights)
        err = float(np.max(np.abs(got_k.weights - ref_w))) / 1e-10
        worst = max(worst, err)
        if err > 1.0:
            failures.append(f"kernel_power h={power} err-ratio={err:.3g}")
        if got_k.min_offset != power * kern.min_offset:
            failures.append(f"kernel_power h={power} offset {got_k.min_offset} != {power * kern.min_offset}")
        steps = int(rng.integers(1, 6))
        span = (len(weights) - 1) * steps
        n = int(rng.integers(span + 1, span + 64))
        row = GridRow(time_index=steps, col_offset=int(rng.integers(-5, 6)), values=rng.uniform(0.0, 1.0, size=n))
        got_row = apply_linear_steps(row, kern, steps, direction=-1)
        ref_vals = row.values
        for _ in range(steps):
            out = np.zeros(len(ref_vals) - len(weights) + 1)
            for w_i, w in enumerate(weights):
                out += w * ref_vals[w_i: w_i + len(out)]
            ref_vals = out
        err = float(np.max(np.abs(got_row.values - ref_vals))) / max(1.0, float(np.max(np.abs(ref_vals)))) / 1e-9
        worst = max(worst, err)
        if err > 1.0:
            failures.append(f"apply_linear_steps n={n} h={steps} err-ratio={err:.3g}")
    return worst, failures


def _suite_european(rng, trials, max_steps):
    """cli.py:349-366: fast vs baseline, one batched call each."""
    hi = max(64, min(max_steps, 65536))
    specs = [_with_steps(_draw_spec(rng, moneyness_band=3.0), int(rng.integers(64, hi + 1))) for _ in range(trials)]
    if not specs:
        return 0.0, []
    fast = _batch(_native.KIND_EURO, specs, _native.METHOD_FAST).price
    base = _batch(_native.KIND_EURO, specs, _native.METHOD_BASELINE).price
    worst, failures = 0.0, []
    for s, f, b in zip(specs, fast, base):
        err = _rel_err(f, b, s.spot) / 1e-8
        worst = max(worst, err)
        if err > 1.0:
            failures.append(f"err-ratio={err:.3g} {_spec_line(s)}")
    return worst, failures


def _suite_american(rng, trials, max_steps):
    """cli.py:369-400: fast vs baseline American call, dominance over the European."""
    hi = max(64, min(max_steps, 4096))
    specs = [_with_steps(_draw_spec(rng, moneyness_band=3.0), int(rng.integers(64, hi + 1))) for _ in range(trials)]
    if not specs:
        return 0.0, []
    fast = _batch(_native.KIND_CALL, specs, _native.METHOD_FAST)
    base = _batch(_native.KIND_CALL, specs, _native.METHOD_BASELINE)
    euro = _batch(_native.KIND_EURO, specs, _native.METHOD_BASELINE).price
    worst, failures = 0.0, []
    for i, s in enumerate(specs):
        err = _rel_err(fast.price[i], base.price[i], s.spot) / 1e-8
        worst = max(worst, err)
        if err > 1.0:
            failures.append(f"price err-ratio={err:.3g} {_spec_line(s)}")
        bt, bc = base.boundary(i)
        brow = dict(zip(bt.tolist(), bc.tolist()))
        for t, col in zip(*map(lambda a: a.tolist(), fast.boundary(i))):
            if brow[t] != col:
                failures.append(f"boundary mismatch at row {t}: fast={col} baseline={brow[t]} {_spec_line(s)}")
                break
        if base.price[i] < euro[i] - 1e-12:
            failures.append(f"american {base.price[i]!r} < european {euro[i]!r} {_spec_line(s)}")
    return worst, failures


def check_boundary_lemmas(spec: OptionSpec) -> str | None:
    """The six boundary lemmas (cli.py:416-484) on a full device grid."""
    n = spec.steps
    result = baseline_american_call(spec, keep_grid=True)
    rows, masks = result.rows, result.exercise_masks
    params = derive_binomial_params(spec)
    dt = params.step_years
    floor_shift = None
    if spec.rate > 0.0 and spec.dividend_yield > 0.0:
        ratio = math.expm1(spec.rate * dt) / math.expm1(spec.dividend_yield * dt)
        floor_shift = (math.log(spec.strike / spec.spot) + math.log(ratio)
                       - (spec.rate - spec.dividend_yield) * dt) / (2.0 * spec.volatility * math.sqrt(dt))
    bounds = np.empty(n + 1, dtype=np.int64)
    for i in range(n + 1):
        mask = masks[i]
        if mask.any():
            first = int(np.argmax(mask))
            if not mask[first:].all():
                return f"(a) row {i}: green run not a suffix"
            bounds[i] = first
        else:
            bounds[i] = i + 1
    for i in range(n):
        below, here = masks[i + 1], masks[i]
        if i < n - 1 and np.any(below[: i + 1] & ~here):
            return f"(b) row {i}: green below without green above"
        if np.any(~below[1: i + 2] & here):
            return f"(c) row {i}: red diagonal below a green cell"
    for i in range(1, n - 1):
        if np.any(rows[i][:i] < rows[i + 2][1: i + 1] - 1e-12):
            return f"(d) row {i}: two-step decay violated"
    for i in range(n):
        if bounds[i] < bounds[i + 1] - 1 or (i < n - 1 and bounds[i] > bounds[i + 1]):
            return f"(e) rows {i},{i + 1}: boundary step {bounds[i]} vs {bounds[i + 1]}"
    if floor_shift is not None:
        for i in range(n):
            if bounds[i] <= i and bounds[i] < i / 2.0 + floor_shift - 1e-9:
                return f"(f) row {i}: green at {bounds[i]} below floor {i / 2.0 + floor_shift:.6g}"
    return None


def _suite_lemmas(rng, trials, max_steps):
    """cli.py:403-413."""
    failures = []
    hi = max(16, min(max_steps, 512))
    for _ in range(trials):
        spec = _with_steps(_draw_spec(rng), int(rng.integers(16, hi + 1)))
        bad = check_boundary_lemmas(spec)
        if bad:
            failures.append(f"{bad} {_spec_line(spec)}")
    return 0.0, failures


def _put_specs(rng, trials, max_steps):
    hi = max(64, min(max_steps, 2048))
    out = []
    while len(out) < trials:
        spec = _with_steps(_draw_spec(rng, moneyness_band=3.0), int(rng.integers(64, hi + 1)))
        try:
            disc = discretize_bsm(spec)
        except (StabilityError, DomainError):
            continue
        out.append((spec, disc))
    return out


def _suite_bsm_theorems(rng, trials, max_steps):
    """cli.py:487-533: weight identity, boundary step / monotonicity theorems."""
    pairs = _put_specs(rng, trials, max_steps)
    if not pairs:
        return 0.0, []
    worst, failures = 0.0, []
    base = _batch(_native.KIND_PUT, [s for s, _ in pairs], _native.METHOD_BASELINE)
    for i, (spec, disc) in enumerate(pairs):
        total = disc.coef_down + disc.coef_mid + disc.coef_up
        ident = 1.0 - disc.omega * disc.d_tau
        err = abs(total - ident) / (4.0 * np.spacing(max(abs(ident), 1.0)))
        worst = max(worst, err)
        if err > 1.0:
            failures.append(f"weight identity off by {total - ident!r} {_spec_line(spec)}")
        _, cols = base.boundary(i)
        seen, prev = False, None
        for col in cols.tolist():
            if col == NO_GREEN:
                seen = True
                continue
            if seen:
                failures.append(f"boundary reappeared after leaving the window {_spec_line(spec)}")
                break
            if prev is not None and not 0 <= prev - col <= 1:
                failures.append(f"boundary step {prev} -> {col} {_spec_line(spec)}")
                break
            prev = int(col)
    return worst, failures


def _suite_bsm_oracle(rng, trials, max_steps):
    """cli.py:536-585: fast vs baseline put, payoff dominance of the handoff rows."""
    pairs = _put_specs(rng, trials, max_steps)
    if not pairs:
        return 0.0, []
    worst, failures = 0.0, []
    base = _batch(_native.KIND_PUT, [s for s, _ in pairs], _native.METHOD_BASELINE)
    for i, (spec, disc) in enumerate(pairs):
        fast = fast_put_bsm(spec, record_rows=True)
        err = _rel_err(fast.price, base.price[i], spec.spot) / 1e-8
        worst = max(worst, err)
        if err > 1.0:
            failures.append(f"price err-ratio={err:.3g} {_spec_line(spec)}")
        bt, bc = base.boundary(i)
        brow = dict(zip(bt.tolist(), bc.tolist()))
        for t, col in fast.boundaries.as_dict().items():
            ref = brow[int(t)]
            if ref != NO_GREEN and ref != col:
                failures.append(f"boundary mismatch at row {t}: fast={col} baseline={ref} {_spec_line(spec)}")
                break
        if fast.rows:
            for t, row in fast.rows.items():
                cols = np.arange(row.first_col, row.last_col + 1)
                payoff = np.maximum(1.0 - np.exp(cols * disc.d_s), 0.0)
                if np.any(row.values < payoff - 1e-12):
                    failures.append(f"payoff dominance violated at row {t} {_spec_line(spec)}")
                    break
        floor = max(bsm_green_value(disc, disc.k_star), 0.0) * spec.strike
        if base.price[i] < floor - 1e-12 * spec.strike:
            failures.append(f"apex {base.price[i]!r} below payoff floor {floor!r} {_spec_line(spec)}")
    return worst, failures


SUITES = (
    ("fft-engine", _suite_fft),
    ("european-oracle", _suite_european),
    ("american-oracle", _suite_american),
    ("binomial-lemmas", _suite_lemmas),
    ("bsm-theorems", _suite_bsm_theorems),
    ("bsm-oracle", _suite_bsm_oracle),
)


def run_suites(reps: int = 25, steps: int = 1024, seed: int = 0, out=sys.stdout) -> int:
    """cmd_verify (cli.py:598-616): exit code 1 if any suite failed."""
    if reps < 0:
        raise ValidationError("reps", "trials must be >= 0")
    if reps == 0:
        return 0
    if steps < 64:
        raise ValidationError("steps", "verification needs steps >= 64")
    failed = False
    for index, (name, suite) in enumerate(SUITES):
        rng = np.random.default_rng([seed, index])
        worst, failures = suite(rng, reps, steps)
        status = "FAIL" if failures else "PASS"
        print(f"{name:<17} {status}  worst-error/tolerance {worst:.3e}  trials {reps}", file=out)
        for line in failures:
            print(f"  {line}", file=out)
        failed = failed or bool(failures)
    return 1 if failed else 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="randomized oracle and invariant suites on the GPU")
    ap.add_argument("--steps", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--reps", type=int, default=25)
    args = ap.parse_args(argv)
    return run_suites(args.reps, args.steps, args.seed)


if __name__ == "__main__":
    sys.exit(main())
