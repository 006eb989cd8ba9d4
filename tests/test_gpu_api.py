"""GPU parity of the drop-in Python API (the reference's own entry points and
exported sub-operators) against golden vectors produced by the reference.

Prices: |d| <= 1e-9 max(|ref|, K); rescaled put rows (values in [0, 1]) and
call rows: |d| <= 1e-9 max(1, K); composed kernels: |d| <= 1e-12 max|W|
(the reference's own FFT round-off is ~1e-16 max|W|); boundaries equal except
at a tie certified by the reference's own margins (conftest.boundary_check)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN, boundary_check, golden, price_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    return np.load(os.path.join(GOLDEN, "ops.npz"))


def test_kernel_power_and_apply_linear_steps(ops):
    import paper_2303_02317_b200 as fl

    for k in range(int(ops["n_kp"])):
        w, off, h = ops[f"kp{k}_w"], int(ops[f"kp{k}_off"]), int(ops[f"kp{k}_h"])
        kern = fl.Kernel(w, off)
        got = fl.kernel_power(kern, h)
        ref = ops[f"kp{k}_out"]
        assert got.min_offset == h * off
        assert got.weights.shape == ref.shape
        assert np.max(np.abs(got.weights - ref)) <= 1e-12 * np.max(np.abs(ref)), (k, h)
        row = fl.GridRow(5000, 3, ops[f"kp{k}_row"])
        r = fl.apply_linear_steps(row, kern, h)
        ref_r = ops[f"kp{k}_als"]
        assert r.col_offset == int(ops[f"kp{k}_als_off"]) and r.time_index == 5000 + h
        assert np.max(np.abs(r.values - ref_r)) <= 1e-12 * max(1.0, np.max(np.abs(ref_r))), (k, h)


def test_apply_linear_steps_errors():
    import paper_2303_02317_b200 as fl

    k = fl.Kernel(np.array([0.5, 0.5]), 0)
    with pytest.raises(fl.InsufficientWidthError):
        fl.apply_linear_steps(fl.GridRow(0, 0, np.ones(3)), k, 5)
    with pytest.raises(fl.ValidationError):
        fl.apply_linear_steps(fl.GridRow(0, 0, np.ones(3)), k, -1)
    out = fl.apply_linear_steps(fl.GridRow(5, 0, np.array([1.0, 2.0, 4.0])), k, 1, direction=-1)
    assert out.time_index == 4 and out.col_offset == 0
    assert np.allclose(out.values, [1.5, 3.0], rtol=0, atol=1e-15)


def _close_rows(got, ref, scale):
    return got.shape == ref.shape and (got.size == 0 or np.max(np.abs(got - ref)) <= 1e-9 * scale)


def test_solve_bsm_trapezoid(ops):
    import paper_2303_02317_b200 as fl
    from paper_2303_02317_b200 import _native

    for k in range(int(ops["n_pt"])):
        cd, cm, cu, ds = ops[f"pt{k}_coef"]
        f, h = int(ops[f"pt{k}_f"]), int(ops[f"pt{k}_h"])
        kp, seg = _native.put_trapezoid(cd, cm, cu, ds, 128, f, ops[f"pt{k}_seg"], h)
        kp_ref, ref = int(ops[f"pt{k}_kp"]), ops[f"pt{k}_out"]
        ok, _, why = boundary_check(2, 1.0, [0], [kp], [0], [kp_ref], ops[f"pt{k}_marg"][None, :])
        assert ok, (k, why)
        # rows cover columns kp+1 .. f+len-h: compare the columns both cover
        d = kp - kp_ref
        got, want = (seg[max(0, -d):], ref[max(0, d):])
        assert _close_rows(got, want, 1.0), (k, np.max(np.abs(got - want)))
        # through the drop-in signature
        disc = fl.BsmDiscretization(0, 0.0, 0.0, 0.0, ds, 0, 0.4, cd, cm, cu)
        st = fl.PutRowState(int(ops[f"pt{k}_t"]), f, fl.GridRow(int(ops[f"pt{k}_t"]), f + 1, ops[f"pt{k}_seg"]))
        nxt = fl.solve_bsm_trapezoid(disc, st, h)
        assert nxt.time_index == st.time_index + h and nxt.boundary == kp
        assert nxt.segment.first_col == kp + 1


def test_solve_bsm_trapezoid_errors():
    import paper_2303_02317_b200 as fl

    disc = fl.discretize_bsm(fl.OptionSpec(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024))
    st = fl.initial_row(disc)
    with pytest.raises(fl.GeometryError):
        fl.solve_bsm_trapezoid(disc, st, 0)
    with pytest.raises(fl.GeometryError):
        fl.solve_bsm_trapezoid(disc, st, len(st.segment))
    with pytest.raises(fl.ValidationError):
        fl.solve_bsm_trapezoid(disc, st, 8, base_cutoff=0)


def test_solve_trapezoid(ops):
    import paper_2303_02317_b200 as fl

    for k in range(int(ops["n_ct"])):
        S, K, R, Y, V, E, T = ops[f"ct{k}_spec"]
        spec = fl.OptionSpec(S, K, R, Y, V, E, int(T))
        i, j, h = int(ops[f"ct{k}_i"]), int(ops[f"ct{k}_j"]), int(ops[f"ct{k}_h"])
        prob = fl.TrapezoidProblem(i, j, h, fl.GridRow(i, 0, ops[f"ct{k}_run"]))
        st = fl.solve_trapezoid(spec, prob)
        jp_ref, ref = int(ops[f"ct{k}_jp"]), ops[f"ct{k}_out"]
        assert st.time_index == i - h
        # first-green columns jp+1 (boundary_check's call convention)
        ok, _, why = boundary_check(1, K, [0], [st.boundary + 1], [0], [jp_ref + 1], ops[f"ct{k}_marg"][None, :])
        assert ok, (k, why)
        # rows cover columns first_col .. jp: compare the columns both cover
        m = min(st.boundary, jp_ref) + 1
        got, want = st.segment.values[:m], ref[:m]
        assert _close_rows(got, want, max(1.0, K)), (k, np.max(np.abs(got - want)))


def test_single_spec_pricers_match_golden():
    """fast_* / baseline_* through the reference signatures on the edge set."""
    import paper_2303_02317_b200 as fl

    for name, method in (("edge_fast", "fast"), ("edge_baseline", "baseline")):
        g = golden(name)
        for i in range(g.n):
            spec = fl.OptionSpec(*g.args(i))
            kind = int(g.kind[i])
            ek = str(g.err_kind[i])
            try:
                if kind == 0:
                    p = fl.fast_european(spec) if method == "fast" else fl.baseline_european(spec)
                    series = None
                elif kind == 1:
                    r = fl.fast_american_call(spec) if method == "fast" else fl.baseline_american_call(spec)
                    p, series = r.price, r.boundaries
                else:
                    r = fl.fast_put_bsm(spec) if method == "fast" else fl.baseline_put_fd(spec)
                    p, series = r.price, r.boundaries
            except (fl.PricingError, ValueError) as e:
                assert type(e).__name__ == ek, (name, i, type(e).__name__, ek)
                fld = getattr(e, "field", getattr(e, "weight", ""))
                assert (fld or "") == str(g.err_field[i]), (name, i, fld, g.err_field[i])
                continue
            assert ek == "", (name, i, ek)
            assert price_close(p, g.price[i], g.K[i]), (name, i, p, g.price[i])
            if series is not None:
                t, c = g.boundary(i)
                assert np.array_equal(series.times, t), (name, i)
                assert np.array_equal(series.columns, c), (name, i)


def test_batch_helpers():
    import paper_2303_02317_b200 as fl

    g = golden("c3_fast")
    sl = slice(0, 32)
    price, status = fl.price_put_batch(g.S[sl], g.K[sl], g.R[sl], g.V[sl], g.E[sl], g.T[sl])
    assert np.all(status == 0)
    for i in range(32):
        assert price_close(price[i], g.price[i], g.K[i])


@pytest.fixture(scope="module")
def api():
    return np.load(os.path.join(GOLDEN, "api.npz"))


def test_keep_grid(api):
    import paper_2303_02317_b200 as fl

    for k in range(int(api["n_g"])):
        S, K, R, Y, V, E, T = api[f"g{k}_spec"]
        spec = fl.OptionSpec(S, K, R, Y, V, E, int(T))
        r = fl.baseline_american_call(spec, keep_grid=True)
        assert price_close(r.price, float(api[f"g{k}_price"]), K)
        assert np.array_equal(r.boundaries.columns, api[f"g{k}_cols"]), k
        rows = np.concatenate(r.rows)
        ref = api[f"g{k}_rows"]
        assert rows.shape == ref.shape
        assert np.max(np.abs(rows - ref)) <= 1e-9 * max(1.0, K), k
        assert np.array_equal(np.concatenate(r.exercise_masks).astype(np.uint8), api[f"g{k}_masks"]), k
        assert len(r.rows) == int(T) + 1 and all(len(x) == i + 1 for i, x in enumerate(r.rows))


def test_baseline_record_rows(api):
    import paper_2303_02317_b200 as fl

    for k in range(int(api["n_b"])):
        S, K, R, Y, V, E, T = api[f"b{k}_spec"]
        spec = fl.OptionSpec(S, K, R, Y, V, E, int(T))
        times = api[f"b{k}_times"].tolist()
        r = fl.baseline_put_fd(spec, 0.4, int(T), record_rows=tuple(times) + (0, int(T) + 5))
        assert price_close(r.price, float(api[f"b{k}_price"]), K)
        assert np.array_equal(r.boundaries.columns, api[f"b{k}_cols"]), k
        assert sorted(r.rows) == times
        vals = np.concatenate([r.rows[t].values for t in times])
        assert [r.rows[t].col_offset for t in times] == api[f"b{k}_offs"].tolist()
        assert np.max(np.abs(vals - api[f"b{k}_vals"])) <= 1e-12, k


def test_fast_record_rows(api):
    import paper_2303_02317_b200 as fl

    for k in range(int(api["n_f"])):
        S, K, R, Y, V, E, T = api[f"f{k}_spec"]
        spec = fl.OptionSpec(S, K, R, Y, V, E, int(T))
        r = fl.fast_put_bsm(spec, 0.4, base_cutoff=int(api[f"f{k}_cut"]), record_rows=True)
        assert price_close(r.price, float(api[f"f{k}_price"]), K)
        assert np.array_equal(r.boundaries.times, api[f"f{k}_times"])
        assert np.array_equal(r.boundaries.columns, api[f"f{k}_cols"])
        ts = sorted(r.rows)
        assert ts == api[f"f{k}_rtimes"].tolist()
        assert [r.rows[t].col_offset for t in ts] == api[f"f{k}_roffs"].tolist()
        assert [len(r.rows[t]) for t in ts] == api[f"f{k}_rlens"].tolist()
        vals = np.concatenate([r.rows[t].values for t in ts])
        assert np.max(np.abs(vals - api[f"f{k}_rvals"])) <= 1e-9, k


def test_fft_and_convolve(api):
    import paper_2303_02317_b200 as fl

    for n in (1, 8, 1024, 4096):
        x = api[f"fft{n}_x"]
        f = fl.fft_forward(x)
        assert np.max(np.abs(f - api[f"fft{n}_f"])) <= 1e-12 * max(1.0, np.max(np.abs(api[f"fft{n}_f"])))
        i = fl.fft_inverse(x)
        assert np.max(np.abs(i - api[f"fft{n}_i"])) <= 1e-12 * max(1.0, np.max(np.abs(api[f"fft{n}_i"])))
        assert np.max(np.abs(fl.fft_inverse(fl.fft_forward(x)) - x)) <= 1e-12  # round trip (test_fft.py)
    for a, b in [(5, 3), (300, 17), (1000, 1000)]:
        z = fl.convolve(api[f"conv{a}_{b}_x"], api[f"conv{a}_{b}_y"])
        ref = api[f"conv{a}_{b}_z"]
        assert z.dtype == np.float64 and z.shape == ref.shape
        assert np.max(np.abs(z - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    assert np.allclose(fl.convolve(np.array([1.0, 1.0]), np.array([1.0, 1.0])), [1.0, 2.0, 1.0], atol=1e-15)


def test_european_approximations(api):
    import paper_2303_02317_b200 as fl

    for row in api["approx"]:
        S, K, R, Y, V, E, T, g_ref, c_ref = row
        spec = fl.OptionSpec(S, K, R, Y, V, E, int(T))
        for fn, ref in ((fl.gaussian_approx_european, g_ref), (fl.closed_form_european, c_ref)):
            if np.isnan(ref):
                with pytest.raises(fl.DomainError):
                    fn(spec)
            else:
                assert price_close(fn(spec), ref, K), (fn.__name__, row)


def test_batch_device_bytes():
    """fl_batch_device_bytes: the device footprint of a prepared batch (the
    per-chain arenas dominate) is positive and grows with T."""
    from paper_2303_02317_b200 import _native

    fp = []
    for T in (1024, 8192):
        db = _native.DeviceBatch(np.full(4, 2, dtype=np.int8), np.full(4, 100.0), np.full(4, 100.0),
                                 np.full(4, 0.05), np.zeros(4), np.full(4, 0.3), np.full(4, 365.0),
                                 np.full(4, T, dtype=np.int64))
        db.run()
        db.fetch()
        fp.append(db.device_bytes())
    assert 0 < fp[0] < fp[1], fp


def test_generic_kernel_power_and_steps_vs_oracle():
    """Kernels beyond the pricers' stencils (fft.py:244-260): more taps,
    negative weights, zero taps -- composed on the device (fl_kernel_power)
    and checked against the oracle's restatement of the reference (numpy
    spectrum power / two-tap closed form) and naive repeated convolution."""
    import paper_2303_02317_b200 as fl
    from oracle import port

    rng = np.random.default_rng(77)
    # (sum |w| <= 1: the spectral route's absolute error scales with max |P(e^it)|^h,
    # in the reference as here)
    cases = [np.array([0.5, -0.1, 0.3]), np.array([-0.4, 0.55]), np.array([0.0, 0.8]), np.array([0.7, 0.0]),
             np.array([0.0, 0.3, 0.0, 0.5, 0.0]), np.array([0.2]), np.array([0.0, 0.0])]
    for _ in range(12):
        taps = int(rng.integers(2, 7))
        w = rng.uniform(-0.2, 1.0, taps)
        cases.append(w / (np.abs(w).sum() * rng.uniform(1.0, 1.3)))
    for w in cases:
        for h in (2, 5, 31, 200):
            got = fl.kernel_power(fl.Kernel(w, -1), h)
            assert got.min_offset == -h and len(got) == h * (len(w) - 1) + 1
            acc = np.array([1.0])
            for _ in range(h):
                acc = np.convolve(acc, w)
            assert np.max(np.abs(got.weights - acc)) <= 1e-10, (w, h)
            if np.count_nonzero(w) and len(w) > 1:
                ref = port.kernel_power(w, h)
                assert np.max(np.abs(got.weights - ref)) <= 1e-10 * max(1.0, np.max(np.abs(ref))), (w, h)
            # exact zeros where a zero end tap forces them (fft.py:176-183)
            nz = np.nonzero(w)[0]
            if nz.size:
                assert np.all(got.weights[:h * nz[0]] == 0.0) and np.all(got.weights[h * nz[-1] + 1:] == 0.0)
        row = fl.GridRow(3, 7, rng.uniform(0.5, 1.5, 400))
        h = 9
        out = fl.apply_linear_steps(row, fl.Kernel(w, -1), h)
        ref = port.valid_corr(row.values, _naive_power(w, h))
        assert out.col_offset == row.col_offset + h and out.time_index == row.time_index + h
        assert np.max(np.abs(out.values - ref)) <= 1e-10 * max(1.0, np.max(np.abs(ref))), w


def _naive_power(w, h):
    acc = np.array([1.0])
    for _ in range(h):
        acc = np.convolve(acc, w)
    return acc


def test_short_linear_jump_keeps_exact_zeros():
    """apply_linear_steps for h <= 64 runs the composed weights directly: a run
    of zeros stays exactly zero, as in the device trapezoid (the reference
    test test_american.py:96-115 compares the two with rtol only)."""
    import paper_2303_02317_b200 as fl

    vals = np.concatenate([np.zeros(120), np.linspace(1e-3, 5.0, 80)])
    k = fl.Kernel(np.array([0.49, 0.5]), 0)
    out = fl.apply_linear_steps(fl.GridRow(100, 0, vals), k, 48, direction=-1)
    assert np.all(out.values[:120 - 48] == 0.0)
    ref = _naive_power(k.weights, 48)
    exp = np.array([ref @ vals[i:i + len(ref)] for i in range(len(vals) - len(ref) + 1)])
    assert np.max(np.abs(out.values - exp)) <= 1e-13 * np.max(exp)


def test_custom_binomial_params():
    """Caller-supplied BinomialParams (binomial.py:80/161, american.py:428):
    the lattice pricers use them (fl_price_batch_ex) instead of the spec's."""
    import paper_2303_02317_b200 as fl
    from oracle import port

    spec = fl.OptionSpec(100.0, 95.0, 0.03, 0.05, 0.25, 180, 2048)
    other = fl.OptionSpec(100.0, 95.0, 0.04, 0.02, 0.31, 200, 2048)
    p = fl.derive_binomial_params(other)
    pd = {"wd": p.weight_down, "wu": p.weight_up, "lu": p.log_up}
    ref = port.euro_fast(spec.spot, spec.strike, spec.rate, spec.dividend_yield, spec.volatility,
                         spec.days_to_expiry, spec.steps, p=pd)
    assert price_close(fl.fast_european(spec, p), ref, spec.strike)
    assert price_close(fl.baseline_european(spec, p), ref, spec.strike)
    assert not price_close(fl.fast_european(spec), ref, spec.strike)
    base = fl.baseline_american_call(spec, p)
    fast = fl.fast_american_call(spec, p)
    assert price_close(fast.price, base.price, spec.strike)
    assert not price_close(fl.fast_american_call(spec).price, base.price, spec.strike)
    grid = fl.baseline_american_call(spec.__class__(*[getattr(spec, f) for f in (
        "spot", "strike", "rate", "dividend_yield", "volatility", "days_to_expiry")], 64), p, keep_grid=True)
    assert np.isfinite(grid.price)
