"""Generate golden vectors by running the REFERENCE itself (this container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the unmodified reference package ``fftlattice`` from
/root/reference/pkg/src, prices seeded batches drawn by
``paper_2303_02317_b200.workloads`` (the BASELINE.json configs, some reduced in
size) plus hand-picked edge cases, and writes ``tests/golden/*.npz``.  The GPU
box has no /root/reference: tests there read only these committed fixtures.
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import fftlattice as fl  # noqa: E402  (the reference)

from paper_2303_02317_b200.workloads import (  # noqa: E402
    KIND_CALL, KIND_EURO, KIND_PUT, Batch, draw_config,
)

ERR_KINDS = ["ValidationError", "StabilityError", "DomainError", "GeometryError",
             "NumericalIntegrityError", "InsufficientWidthError", "UnsupportedCombinationError"]


def run_ref(kind, spec, method="fast"):
    """(price, times, cols, err_kind, err_field) from the reference."""
    try:
        if kind == KIND_EURO:
            p = fl.fast_european(spec) if method == "fast" else fl.baseline_european(spec)
            t, c = np.zeros(0, np.int64), np.zeros(0, np.int64)
        elif kind == KIND_CALL:
            r = fl.fast_american_call(spec) if method == "fast" else fl.baseline_american_call(spec)
            p, t, c = r.price, r.boundaries.times, r.boundaries.columns
        else:
            r = fl.fast_put_bsm(spec, 0.4) if method == "fast" else fl.baseline_put_fd(spec, 0.4)
            p, t, c = r.price, r.boundaries.times, r.boundaries.columns
        return float(p), np.asarray(t, np.int64), np.asarray(c, np.int64), "", ""
    except (fl.PricingError, ValueError) as e:
        # ValueError: the reference's own math-domain failure (zero strike on
        # the American junction path, american.py:403) is mirrored too.
        fld = getattr(e, "field", getattr(e, "weight", ""))
        return math.nan, np.zeros(0, np.int64), np.zeros(0, np.int64), type(e).__name__, fld or ""


# --- boundary margins -------------------------------------------------------
# north_star allows a boundary index to differ from the reference's only "at
# ties within tolerance".  To check that on the device without the reference,
# the goldens carry, for every boundary record the reference produced with a
# leaf strip, the reference's own  lin - exercise  at the 7 cells around its
# boundary on that record's row (cells b-3 .. b+3, b = last exercise column for
# the put, last continuation column for the call).  They are computed by
# re-running the reference's strip sweep (unmodified numba kernel) for
# height-1 rows on a copy and evaluating the last row with the kernel's own
# expression and evaluation order (_accel.py:232 put, :148-149 call), so they
# are the reference's bits.  Put margins are in units of K (the put grid is
# normalised by the strike), call margins in currency units; NaN where the
# record was not produced by a strip (payoff row, junction row, baseline
# dispatch) -- those records get no slack.
from fftlattice import _accel as _ref_accel  # noqa: E402
from fftlattice import bsm as _ref_bsm  # noqa: E402

NMARG = 7
_MARG: dict = {}
_orig_strip_advance = _ref_bsm._strip_advance
_orig_binomial_sweep = _ref_accel.binomial_strip_sweep


def _strip_advance_margins(ctx, time_index, boundary, seg, height):
    kb, out = _orig_strip_advance(ctx, time_index, boundary, seg, height)
    disc = ctx.disc
    cd, cm, cu = disc.coef_down, disc.coef_mid, disc.coef_up
    f = boundary
    hi = f + seg.shape[0]
    lo = f - 2 * height - 1
    payoff = _ref_bsm._payoff_slice(disc, lo, hi)
    arr = np.empty(hi - lo + 1, dtype=np.float64)
    arr[: f - lo + 1] = payoff[: f - lo + 1]
    arr[f - lo + 1:] = seg
    if height > 1:
        _ref_accel.bsm_strip_sweep(arr, payoff, lo, height - 1, cd, cm, cu)
    m = np.full(NMARG, np.nan)
    for d in range(-(NMARG // 2), NMARG // 2 + 1):
        k = kb + d
        if lo + height <= k <= hi - height:
            left, cur, right = arr[k - 1 - lo], arr[k - lo], arr[k + 1 - lo]
            lin = cm * cur + cu * right + cd * left
            m[d + NMARG // 2] = lin - payoff[k - lo]
    _MARG[time_index + height] = m
    return kb, out


def _binomial_sweep_margins(values, e2, lo, top_row, boundary, height, spot, strike, wd, wu, log_up):
    buf = values.copy()
    jr = int(_orig_binomial_sweep(values, e2, lo, top_row, boundary, height, spot, strike, wd, wu, log_up))
    j1 = boundary
    if height > 1:
        j1 = int(_orig_binomial_sweep(buf, e2, lo, top_row, boundary, height - 1, spot, strike, wd, wu, log_up))
    m = np.full(NMARG, np.nan)
    parent = top_row - (height - 1)
    child = parent - 1
    if j1 >= lo:
        top = j1 if j1 < child else child
        base_child = spot * math.exp((2 * lo - child) * log_up)
        base_parent = spot * math.exp((2 * lo - parent) * log_up)
        for d in range(-(NMARG // 2), NMARG // 2 + 1):
            c = jr + d
            if lo <= c <= top:
                vr = buf[c + 1 - lo] if c + 1 <= j1 else base_parent * e2[c + 1 - lo] - strike
                lin = wd * buf[c - lo] + wu * vr
                grn = base_child * e2[c - lo] - strike
                m[d + NMARG // 2] = lin - grn
    _MARG[top_row - height] = m
    return jr


_ref_bsm._strip_advance = _strip_advance_margins
_ref_accel.binomial_strip_sweep = _binomial_sweep_margins


def run_ref_marg(kind, spec, method="fast"):
    """run_ref plus the per-record boundary margins (n_rec x NMARG)."""
    _MARG.clear()
    p, t, c, ek, ef = run_ref(kind, spec, method)
    marg = np.full((len(t), NMARG), np.nan)
    if kind != KIND_EURO and method == "fast":
        for r, tm in enumerate(t.tolist()):
            if tm in _MARG:
                marg[r] = _MARG[tm]
    return p, t, c, ek, ef, marg


def _run_one(args):
    kind, spec, method = args
    return run_ref_marg(kind, spec, method)


def save(name, batch: Batch, method="fast", procs=None):
    """Price ``batch`` with the reference (``procs`` forked workers) and save."""
    import multiprocessing as mp

    t0 = time.time()
    prices, terr, tfld, offs, times, cols, margs = [], [], [], [0], [], [], []
    jobs = [(int(batch.kind[i]), batch.spec(i), method) for i in range(len(batch))]
    procs = procs or int(os.environ.get("GOLDEN_PROCS", os.cpu_count() or 1))
    if procs > 1 and len(jobs) > 8:
        with mp.get_context("fork").Pool(procs) as pool:
            results = pool.map(_run_one, jobs, chunksize=1)
    else:
        results = [_run_one(j) for j in jobs]
    for p, t, c, ek, ef, mg in results:
        prices.append(p); terr.append(ek); tfld.append(ef)
        times.append(t); cols.append(c); offs.append(offs[-1] + len(t)); margs.append(mg)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        kind=batch.kind, S=batch.S, K=batch.K, R=batch.R, Y=batch.Y, V=batch.V,
        E=batch.E, T=batch.T, price=np.asarray(prices), err_kind=np.asarray(terr),
        err_field=np.asarray(tfld), bnd_off=np.asarray(offs, np.int64),
        bnd_times=np.concatenate(times) if times else np.zeros(0, np.int64),
        bnd_cols=np.concatenate(cols) if cols else np.zeros(0, np.int64),
        bnd_marg=np.concatenate(margs) if margs else np.zeros((0, NMARG)),
        method=np.asarray(method),
    )
    print(f"{name}: {len(batch)} options, {time.time() - t0:.1f}s", flush=True)


def from_specs(rows):
    kinds = [r[0] for r in rows]
    specs = [r[1] for r in rows]
    n = len(rows)
    b = Batch(np.asarray(kinds, np.int8), *(np.empty(n) for _ in range(6)), np.empty(n, np.int64))
    for i, s in enumerate(specs):
        b.S[i], b.K[i], b.R[i], b.Y[i] = s.spot, s.strike, s.rate, s.dividend_yield
        b.V[i], b.E[i], b.T[i] = s.volatility, s.days_to_expiry, s.steps
    return b


def edge_cases():
    O = fl.OptionSpec
    rows = [
        # reference KAT specs (test_binomial.py:39-47, test_american.py:38-39, test_bsm.py:30-33)
        (KIND_EURO, O(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024)),
        (KIND_CALL, O(100.0, 90.0, 0.03, 0.07, 0.25, 365, 512)),
        (KIND_CALL, O(150.0, 80.0, 0.09, 0.05, 0.15, 365, 512)),  # junction widening
        (KIND_PUT, O(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024)),
        # dispatch branches
        (KIND_CALL, O(120.0, 100.0, 0.05, 0.0, 0.3, 365, 4096)),   # Y == 0 -> European
        (KIND_CALL, O(100.0, 95.0, 0.04, 0.06, 0.3, 365, 200)),    # T <= cutoff -> baseline
        (KIND_CALL, O(50.0, 200.0, 0.05, 0.03, 0.1, 30, 512)),     # all-red terminal row
        (KIND_CALL, O(100.0, 0.0, 0.05, 0.03, 0.2, 365, 1024)),    # zero strike
        (KIND_CALL, O(200.0, 50.0, 0.01, 0.1, 0.1, 365, 1024)),    # deep ITM, large yield
        (KIND_PUT, O(50.0, 160.0, 0.05, 0.0, 0.2, 365, 16)),       # k* <= -T intrinsic
        (KIND_PUT, O(100.0, 100.0, 0.04, 0.0, 0.25, 180, 200)),    # T <= 2 cutoff -> baseline
        (KIND_PUT, O(140.0, 100.0, 0.03, 0.0, 0.5, 60, 16384)),    # k* > 0 (Appendix C P3)
        (KIND_PUT, O(90.0, 110.0, 0.06, 0.0, 0.35, 500, 16384)),   # k* < 0 (Appendix C P2)
        (KIND_PUT, O(100.0, 100.0, 0.05, 0.0, 0.2, 365, 4096)),
        (KIND_PUT, O(60.0, 100.0, 0.08, 0.0, 0.1, 30, 1000)),      # deep ITM, boundary far down
        (KIND_PUT, O(150.0, 50.0, 0.01, 0.0, 0.6, 730, 2000)),     # far OTM put
        (KIND_EURO, O(100.0, 95.0, 0.03, 0.05, 0.25, 180, 16384)),
        (KIND_CALL, O(100.0, 95.0, 0.03, 0.05, 0.25, 180, 16384)),
        (KIND_CALL, O(120.0, 100.0, 0.04, 0.02, 0.35, 300, 16384)),
        (KIND_CALL, O(80.0, 110.0, 0.02, 0.04, 0.45, 90, 16384)),
        # error parity
        (KIND_PUT, O(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024)),    # fine
        (KIND_PUT, O(200.0, 50.0, 0.05, 0.0, 0.1, 30, 4)),         # DomainError grid nodes
        (KIND_PUT, O(100.0, 0.0, 0.05, 0.0, 0.2, 365, 64)),        # DomainError strike
        (KIND_EURO, O(-1.0, 100.0, 0.05, 0.0, 0.2, 365, 64)),      # ValidationError spot
        (KIND_CALL, O(100.0, 100.0, 0.05, 0.02, 0.0, 365, 64)),    # ValidationError volatility
        (KIND_CALL, O(100.0, 100.0, 0.9, 0.0, 0.01, 365, 4)),      # prob_up out of range
    ]
    # a StabilityError put: search a seeded stream for one
    rng = np.random.default_rng(7)
    while True:
        s = O(float(rng.uniform(50, 200)), float(rng.uniform(50, 200)), float(rng.uniform(0.01, 0.1)),
              0.0, float(rng.uniform(0.1, 0.5)), int(rng.integers(30, 731)), int(rng.integers(64, 1024)))
        try:
            fl.discretize_bsm(s, 0.4)
        except fl.StabilityError:
            rows.append((KIND_PUT, s))
            break
    return from_specs(rows)


def small_random(seed, n, tlo, thi):
    """Random specs (all three kinds) at small T, for full-boundary baseline goldens."""
    rng = np.random.default_rng([seed, 20261019])
    rows = []
    while len(rows) < n:
        kind = int(rng.integers(0, 3))
        T = int(rng.integers(tlo, thi + 1))
        s = fl.OptionSpec(float(rng.uniform(50, 150)), float(rng.uniform(50, 150)),
                          float(rng.uniform(0.01, 0.08)),
                          0.0 if kind == KIND_PUT else float(rng.uniform(0.0, 0.06)),
                          float(rng.uniform(0.1, 0.6)), float(rng.uniform(30, 730)), T)
        try:
            if kind == KIND_PUT:
                fl.discretize_bsm(s, 0.4)
            else:
                fl.derive_binomial_params(s)
        except fl.PricingError:
            continue
        rows.append((kind, s))
    return from_specs(rows)


def stratified_c5(per=2):
    b = draw_config(5)
    idx = []
    for kind in (KIND_EURO, KIND_CALL, KIND_PUT):
        for e in range(10, 17):
            sel = np.nonzero((b.kind == kind) & (b.T == 2 ** e))[0][:per]
            idx.extend(sel.tolist())
    return b.subset(np.asarray(idx))


def ops_cases():
    """Golden vectors for the exported sub-operators the reference tests drive
    directly: kernel_power, apply_linear_steps, solve_bsm_trapezoid,
    solve_trapezoid.  Saved as ops.npz with per-case keys."""
    from fftlattice import american as ref_american

    out = {}
    O = fl.OptionSpec
    rng = np.random.default_rng([99, 20261019])
    # kernel_power / apply_linear_steps on the pricers' own stencils
    put_disc = fl.discretize_bsm(O(100.0, 100.0, 0.05, 0.0, 0.2, 365, 4096), 0.4)
    bp = fl.derive_binomial_params(O(100.0, 95.0, 0.03, 0.05, 0.25, 180, 4096))
    kernels = [("put", np.array([put_disc.coef_down, put_disc.coef_mid, put_disc.coef_up]), -1),
               ("call", np.array([bp.weight_down, bp.weight_up]), 0)]
    k = 0
    for name, w, off in kernels:
        for h in (2, 7, 33, 64, 65, 300, 1000, 5000):
            kern = fl.Kernel(w, off)
            out[f"kp{k}_w"] = w
            out[f"kp{k}_off"] = np.asarray(off)
            out[f"kp{k}_h"] = np.asarray(h)
            out[f"kp{k}_out"] = fl.kernel_power(kern, h).weights
            L = int(rng.integers(len(w) + h * (len(w) - 1), 3 * h * len(w) + 50))
            row = fl.GridRow(5000, 3, rng.uniform(0.0, 1.0, L))
            r = fl.apply_linear_steps(row, kern, h)
            out[f"kp{k}_row"] = row.values
            out[f"kp{k}_als"] = r.values
            out[f"kp{k}_als_off"] = np.asarray(r.col_offset)
            k += 1
    out["n_kp"] = np.asarray(k)
    # solve_bsm_trapezoid: two consecutive stages from the payoff row
    k = 0
    for spec, h0 in [(O(100.0, 100.0, 0.05, 0.0, 0.2, 365, 4096), 700),
                     (O(90.0, 110.0, 0.06, 0.0, 0.35, 500, 16384), 3000),
                     (O(140.0, 100.0, 0.03, 0.0, 0.5, 60, 2048), 100),
                     (O(100.0, 100.0, 0.04, 0.0, 0.25, 180, 1024), 37)]:
        disc = fl.discretize_bsm(spec, 0.4)
        st = fl.initial_row(disc)
        for h in (h0, max(1, h0 // 3)):
            if len(st.segment) < 2 * h:
                break
            _MARG.clear()
            nxt = fl.solve_bsm_trapezoid(disc, st, h)
            out[f"pt{k}_marg"] = _MARG.get(st.time_index + h, np.full(NMARG, np.nan))
            out[f"pt{k}_coef"] = np.array([disc.coef_down, disc.coef_mid, disc.coef_up, disc.d_s])
            out[f"pt{k}_f"] = np.asarray(st.boundary)
            out[f"pt{k}_t"] = np.asarray(st.time_index)
            out[f"pt{k}_seg"] = st.segment.values
            out[f"pt{k}_h"] = np.asarray(h)
            out[f"pt{k}_kp"] = np.asarray(nxt.boundary)
            out[f"pt{k}_out"] = nxt.segment.values
            st = nxt
            k += 1
    out["n_pt"] = np.asarray(k)
    # solve_trapezoid: the first trapezoid after the junction row, and the next one
    k = 0
    for spec in [O(100.0, 95.0, 0.03, 0.05, 0.25, 180, 4096), O(120.0, 100.0, 0.04, 0.02, 0.35, 300, 16384),
                 O(80.0, 110.0, 0.02, 0.04, 0.45, 90, 2048)]:
        p = fl.derive_binomial_params(spec)
        top = fl.top_row_state(spec, p)
        junc = ref_american._junction_row(spec, p, top)
        i, j, vals = junc.time_index, junc.boundary, junc.segment.values
        resid = math.isqrt(spec.steps - 1) + 1
        for _ in range(2):
            if not (i > resid and j >= 0):
                break
            h = min(j + 1, i - resid)
            prob = fl.TrapezoidProblem(i, j, h, fl.GridRow(i, 0, vals))
            _MARG.clear()
            st = fl.solve_trapezoid(spec, prob, p)
            out[f"ct{k}_marg"] = _MARG.get(i - h, np.full(NMARG, np.nan))
            out[f"ct{k}_spec"] = np.array([spec.spot, spec.strike, spec.rate, spec.dividend_yield,
                                           spec.volatility, spec.days_to_expiry, spec.steps], dtype=np.float64)
            out[f"ct{k}_i"] = np.asarray(i)
            out[f"ct{k}_j"] = np.asarray(j)
            out[f"ct{k}_h"] = np.asarray(h)
            out[f"ct{k}_run"] = vals
            out[f"ct{k}_jp"] = np.asarray(st.boundary)
            out[f"ct{k}_out"] = st.segment.values
            i, j, vals = st.time_index, st.boundary, st.segment.values
            k += 1
    out["n_ct"] = np.asarray(k)
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **out)
    print(f"ops: {int(out['n_kp'])} kernel cases, {int(out['n_pt'])} put stages, {int(out['n_ct'])} trapezoids")


def api_cases():
    """Golden vectors for the structural API options the reference tests use:
    keep_grid, record_rows (baseline and fast), fft_forward / fft_inverse /
    convolve.  Saved as api.npz."""
    out = {}
    O = fl.OptionSpec
    rng = np.random.default_rng([98, 20261019])
    k = 0
    for spec in [O(100.0, 90.0, 0.03, 0.07, 0.25, 365, 64), O(150.0, 80.0, 0.09, 0.05, 0.15, 365, 200),
                 O(100.0, 100.0, 0.05, 0.0, 0.2, 365, 33)]:
        r = fl.baseline_american_call(spec, keep_grid=True)
        out[f"g{k}_spec"] = np.array([spec.spot, spec.strike, spec.rate, spec.dividend_yield, spec.volatility,
                                      spec.days_to_expiry, spec.steps])
        out[f"g{k}_price"] = np.asarray(r.price)
        out[f"g{k}_cols"] = r.boundaries.columns
        out[f"g{k}_rows"] = np.concatenate(r.rows)
        out[f"g{k}_masks"] = np.concatenate(r.exercise_masks).astype(np.uint8)
        k += 1
    out["n_g"] = np.asarray(k)
    k = 0
    for spec, steps, rec in [(O(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024), 512, (100, 300, 500)),
                             (O(90.0, 110.0, 0.06, 0.0, 0.35, 500, 300), None, (1, 150, 299, 300))]:
        r = fl.baseline_put_fd(spec, 0.4, steps, record_rows=rec)
        out[f"b{k}_spec"] = np.array([spec.spot, spec.strike, spec.rate, spec.dividend_yield, spec.volatility,
                                      spec.days_to_expiry, spec.steps if steps is None else steps])
        out[f"b{k}_price"] = np.asarray(r.price)
        out[f"b{k}_cols"] = r.boundaries.columns
        ts = sorted(r.rows)
        out[f"b{k}_times"] = np.asarray(ts, dtype=np.int64)
        out[f"b{k}_offs"] = np.asarray([r.rows[t].col_offset for t in ts], dtype=np.int64)
        out[f"b{k}_vals"] = np.concatenate([r.rows[t].values for t in ts])
        k += 1
    out["n_b"] = np.asarray(k)
    k = 0
    for spec, cut in [(O(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024), 32), (O(140.0, 100.0, 0.03, 0.0, 0.5, 60, 4096), 128)]:
        r = fl.fast_put_bsm(spec, 0.4, base_cutoff=cut, record_rows=True)
        out[f"f{k}_spec"] = np.array([spec.spot, spec.strike, spec.rate, spec.dividend_yield, spec.volatility,
                                      spec.days_to_expiry, spec.steps])
        out[f"f{k}_cut"] = np.asarray(cut)
        out[f"f{k}_price"] = np.asarray(r.price)
        out[f"f{k}_times"] = r.boundaries.times
        out[f"f{k}_cols"] = r.boundaries.columns
        ts = sorted(r.rows)
        out[f"f{k}_rtimes"] = np.asarray(ts, dtype=np.int64)
        out[f"f{k}_roffs"] = np.asarray([r.rows[t].col_offset for t in ts], dtype=np.int64)
        out[f"f{k}_rlens"] = np.asarray([len(r.rows[t]) for t in ts], dtype=np.int64)
        out[f"f{k}_rvals"] = np.concatenate([r.rows[t].values for t in ts])
        k += 1
    out["n_f"] = np.asarray(k)
    for n in (1, 8, 1024, 4096):
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        out[f"fft{n}_x"] = x
        out[f"fft{n}_f"] = fl.fft_forward(x)
        out[f"fft{n}_i"] = fl.fft_inverse(x)
    for a, b in [(5, 3), (300, 17), (1000, 1000)]:
        x = rng.standard_normal(a)
        y = rng.standard_normal(b)
        out[f"conv{a}_{b}_x"] = x
        out[f"conv{a}_{b}_y"] = y
        out[f"conv{a}_{b}_z"] = fl.convolve(x, y)
    # European normal-limit approximations (binomial.py:197-296), incl. their DomainErrors
    specs = [O(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024), O(100.0, 95.0, 0.03, 0.05, 0.25, 180, 16384),
             O(120.0, 100.0, 0.04, 0.02, 0.35, 300, 4096), O(80.0, 110.0, 0.02, 0.04, 0.45, 90, 65536),
             O(100.0, 0.0, 0.05, 0.0, 0.2, 365, 64), O(100.0, 300.0, 0.05, 0.0, 0.1, 10, 64),
             O(100.0, 100.0, 0.05, 0.0, 0.2, 365, 2)]
    vals = []
    for spec in specs:
        row = [spec.spot, spec.strike, spec.rate, spec.dividend_yield, spec.volatility, spec.days_to_expiry,
               spec.steps]
        for fn in (fl.gaussian_approx_european, fl.closed_form_european):
            try:
                row.append(fn(spec))
            except fl.DomainError:
                row.append(np.nan)
        vals.append(row)
    out["approx"] = np.asarray(vals)
    np.savez_compressed(os.path.join(HERE, "api.npz"), **out)
    print("api: keep_grid, record_rows, fft cases written")


def batch_case():
    """A portfolio CSV exercising every combination and error column, with the
    reference's own cmd_batch output (cli.py:797-842)."""
    import argparse
    import contextlib
    import io

    from fftlattice import cli

    rows = [
        "european,call,binomial,fast,100,100,0.05,0,0.2,365,1024,",
        "european,call,binomial,baseline,100,95,0.03,0.05,0.25,180,512,",
        "european,call,binomial,gaussian,120,100,0.04,0.02,0.35,300,4096,",
        "european,call,binomial,closed-form,80,110,0.02,0.04,0.45,90,16384,",
        "american,call,binomial,fast,100,90,0.03,0.07,0.25,365,512,",
        "american,call,binomial,baseline,150,80,0.09,0.05,0.15,365,300,",
        "american,put,bsm,fast,100,100,0.05,0,0.2,365,1024,0.4",
        "american,put,bsm,baseline,90,110,0.06,0,0.35,500,400,",
        "american,put,bsm,fast,140,100,0.03,0,0.5,60,4096,0.3",
        "american,put,bsm,fast,100,100,0.05,0,0.2,365,1024,0.9",   # StabilityError -> lambda
        "american,put,bsm,fast,100,100,0.05,0,0.2,365,1024,abc",   # unparsable lambda
        "american,put,bsm,fast,100,100,0.05,0,0.2,365,1024,0",     # lam must be positive
        "american,put,bsm,fast,100,0,0.05,0,0.2,365,64,",          # DomainError -> S
        "american,put,bsm,fast,100,100,0.05,-1,0.2,365,64,",       # ValidationError dividend -> Y
        "american,call,bsm,fast,100,100,0.05,0,0.2,365,64,",       # unsupported combination
        "european,call,binomial,fast,100,100,0.05,0,0.2,365.5,64,",  # E not an int
        "european,call,binomial,fast,-1,100,0.05,0,0.2,365,64,",   # spot
        "european,call,binomial,fast,100,100,0.9,0,0.01,365,4,",   # prob_up -> T? (field prob_up)
        "european,call,binomial,gaussian,100,100,0.05,0,0.2,365,2,",
        "european,call,binomial,closed-form,100,0,0.05,0,0.2,365,64,",
        "american,call,binomial,fast,100,95,0.04,0.06,0.3,365,200,",
        "european,call,binomial,fast,100,100,0.05,0,0.2,365",      # short row
        "european,call,binomial,fast,100,100,0.05,0,0.2,365,64,,x",  # long row
    ]
    text = "style,right,model,method,S,K,R,Y,V,E,T,lambda\n" + "\n".join(rows) + "\n"
    path = os.path.join(HERE, "portfolio.csv")
    with open(path, "w") as fh:
        fh.write(text)
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.cmd_batch(argparse.Namespace(csv=path, parallel=False))
    with open(os.path.join(HERE, "portfolio_ref.csv"), "w") as fh:
        fh.write(buf.getvalue())
    print(f"batch: {len(rows)} rows, reference exit code {rc}")


def bench_case():
    """The reference's own bench CSV (cli.py:653-720) for every method at two
    step counts: its price column is the golden for benchcsv.py."""
    import argparse
    import contextlib
    import io

    from fftlattice import cli

    buf = io.StringIO()
    ns = argparse.Namespace(method=",".join(cli._BENCH_METHODS), steps="300,1024", spot=100.0, strike=100.0,
                            rate=0.05, dividend_yield=0.03, vol=0.2, days=365, lam=0.4, reps=1, csv=None,
                            parallel=False)
    with contextlib.redirect_stdout(buf):
        rc = cli.cmd_bench(ns)
    with open(os.path.join(HERE, "bench_ref.csv"), "w") as fh:
        fh.write(buf.getvalue())
    print(f"bench: reference exit code {rc}")


def verify_case():
    """The reference's own verify output (cli.py:598-616) for a fixed seed."""
    import argparse
    import contextlib
    import io

    from fftlattice import cli

    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.cmd_verify(argparse.Namespace(reps=6, steps=1024, seed=3))
    with open(os.path.join(HERE, "verify_ref.txt"), "w") as fh:
        fh.write(buf.getvalue())
    print(f"verify: reference exit code {rc}")


if __name__ == "__main__":
    which = set(sys.argv[1:])
    want = lambda k: not which or k in which  # noqa: E731
    if want("edge"):
        save("edge_fast", edge_cases(), "fast")
        save("edge_baseline", edge_cases(), "baseline")
    if want("small"):
        sm = small_random(1, 96, 40, 1500)
        save("small_fast", sm, "fast")
        save("small_baseline", sm, "baseline")
    if want("c1"):
        save("c1_fast", draw_config(1), "fast")
    if want("c2"):
        save("c2_fast", draw_config(2), "fast")
    if want("c3"):
        save("c3_fast", draw_config(3), "fast")
    if want("c6"):
        save("c6_fast", draw_config(6, n=256), "fast")  # every timed headline option
    if want("c4"):
        save("c4_fast", draw_config(4), "fast")  # all 64 puts + 64 calls
    if want("c5"):
        save("c5_fast", stratified_c5(per=49), "fast")  # >= 1/64 of every (kind, T) stratum
    if want("ops"):
        ops_cases()
    if want("api"):
        api_cases()
    if want("batch"):
        batch_case()
    if want("verify"):
        verify_case()
    if want("bench"):
        bench_case()
