"""CPU-side tests: the C ABI loads and exports every declared symbol, the
host-side parameter derivation (C++ fl_inspect and the Python model) is
bit-identical to the reference's, status codes map onto the reference
exceptions, seeded workloads are deterministic, sharding is balanced, and
API argument checks raise before any device work.  No GPU needed."""

from __future__ import annotations

import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

from oracle import port


def test_library_exports_every_declared_symbol(native):
    from paper_2303_02317_b200 import _native

    header = open(os.path.join(ROOT, "include", "fftlattice_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|const char\*|int64_t)\s+(fl_\w+)\(", header, re.M))
    assert declared == set(_native.EXPORTED_SYMBOLS), declared ^ set(_native.EXPORTED_SYMBOLS)
    for s in declared:
        assert hasattr(native, s), s
    assert native.fl_version() >= 100


def test_build_flags_target_sm100a():
    from paper_2303_02317_b200 import build

    assert build.ARCH == ["-gencode", "arch=compute_100a,code=sm_100a"]


def _py_derivation(kind, args):
    """(status-kind, tuple of derived constants) from the Python model."""
    import paper_2303_02317_b200 as fl

    spec = fl.OptionSpec(*args)
    try:
        if kind == 2:
            d = fl.discretize_bsm(spec, 0.4)
            return "", (d.coef_down, d.coef_mid, d.coef_up, d.d_s, d.k_star)
        p = fl.derive_binomial_params(spec)
        return "", (p.weight_down, p.weight_up, p.log_up)
    except fl.PricingError as e:
        return type(e).__name__, getattr(e, "field", getattr(e, "weight", None))


@pytest.mark.parametrize("name", ["edge_fast", "small_fast", "c5_fast", "c3_fast", "c2_fast"])
def test_host_derivation_bit_exact(name):
    """C++ (fl_inspect) and Python derivations agree bit for bit with each other
    and with the oracle (which is pinned to the reference)."""
    from paper_2303_02317_b200 import _native

    g = golden(name)
    status, mode, dp, ip = _native.inspect(g.kind, g.S, g.K, g.R, g.Y, g.V, g.E, g.T)
    for i in range(g.n):
        args = g.args(i)
        kind = int(g.kind[i])
        ek, vals = _py_derivation(kind, args)
        if ek:
            err = _native.status_error(int(status[i]))
            assert err is not None and type(err).__name__ == ek, (name, i, ek, hex(status[i]))
            continue
        if status[i] != 0:  # host-decided error the Python model does not raise (e.g. math domain)
            assert str(g.err_kind[i]) != "", (name, i, hex(status[i]))
            continue
        if kind == 2:
            cd, cm, cu, ds, ks = vals
            assert (dp[i, 0], dp[i, 1], dp[i, 2], dp[i, 3], ip[i, 0]) == (cd, cm, cu, ds, ks), (name, i)
            o = port.discretize_put(*args)
            assert (o["cd"], o["cm"], o["cu"], o["d_s"], o["k_star"]) == (cd, cm, cu, ds, ks)
        else:
            wd, wu, lu = vals
            o = port.derive_binomial(*args)
            assert (o["wd"], o["wu"], o["lu"]) == (wd, wu, lu)
            if kind == 1:
                assert (dp[i, 0], dp[i, 1], dp[i, 2]) == (wd, wu, lu), (name, i)
            else:
                assert (dp[i, 0], dp[i, 1], dp[i, 3]) == (wd, wu, lu), (name, i)


def test_call_dispatch_and_boundaries_match_reference_records():
    """Terminal / junction boundaries derived on the host equal the first two
    records of the reference's boundary series (american.py:471-476)."""
    from paper_2303_02317_b200 import _native

    g = golden("c2_fast")
    status, mode, dp, ip = _native.inspect(g.kind, g.S, g.K, g.R, g.Y, g.V, g.E, g.T)
    fg = lambda i, j: port.NO_GREEN if j >= i else j + 1  # noqa: E731
    for i in range(g.n):
        assert status[i] == 0 and mode[i] == 0
        t, c = g.boundary(i)
        n = int(g.T[i])
        rec = dict(zip(t.tolist(), c.tolist()))
        assert rec[n] == fg(n, ip[i, 0])
        assert rec[n - 1] == fg(n - 1, ip[i, 1])


def test_put_dispatch_modes():
    from paper_2303_02317_b200 import _native

    # k* <= -T -> closed price; T <= 2 cutoff -> baseline; else fast; K = 0 -> DomainError
    S = np.array([50.0, 100.0, 100.0, 100.0])
    K = np.array([160.0, 100.0, 100.0, 0.0])
    T = np.array([16, 200, 4096, 64])
    st, mode, _, _ = _native.inspect(2, S, K, 0.05, 0.0, 0.2, 365.0, T)
    assert list(mode[:3]) == [2, 1, 0]
    assert type(_native.status_error(st[3])).__name__ == "DomainError"


def test_put_sliding_strip_flag():
    """The host enables the sliding-frame leaf strip only when an exercise cell
    whose three parents are exercise cells provably stays one: lin - payoff =
    -omega dtau + e^x (1 - A) < -1e-12 for every x <= 0 (fl_put.cu put_leaf,
    fl_strip.cuh put_strip_slide).  Restated here from the reference's grid
    constants (bsm.py:150-229); the drawn rates straddle the cut."""
    from paper_2303_02317_b200 import _native

    rows = [(100.0, 100.0, R, V, 365.0, T) for R in (0.0, 1e-6, 1e-5, 1e-3, 0.05)
            for V in (0.1, 0.3, 0.6) for T in (1024, 4096)]
    S, K, R, V, E, T = (np.array([r[i] for r in rows]) for i in range(6))
    st, mode, _, ip = _native.inspect(2, S, K, R, 0.0, V, E, T.astype(np.int64))
    seen = set()
    for i, r in enumerate(rows):
        d = port.discretize_put(r[0], r[1], r[2], 0.0, r[3], r[4], int(r[5]), 0.4)
        A = d["cd"] * math.exp(-d["d_s"]) + d["cm"] + d["cu"] * math.exp(d["d_s"])
        want = int(d["omega"] * d["d_tau"] - max(0.0, 1.0 - A) > 1e-12)
        assert st[i] == 0 and ip[i, 1] == want, (r, ip[i, 1], want)
        seen.add(want)
    assert seen == {0, 1}


def test_status_error_mapping():
    import paper_2303_02317_b200 as fl
    from paper_2303_02317_b200 import _native

    e = _native.status_error(0x100 | 1)
    assert isinstance(e, fl.ValidationError) and isinstance(e, ValueError) and e.field == "spot"
    e = _native.status_error(0x100 | 8)
    assert e.field == "prob_up"
    e = _native.status_error(0x200 | 1)
    assert isinstance(e, fl.StabilityError) and e.weight == "coef_mid"
    assert isinstance(_native.status_error(0x300 | 1), fl.DomainError)
    assert isinstance(_native.status_error(0x400 | 3), fl.GeometryError)
    assert _native.status_error(0) is None


def test_workloads_deterministic_and_in_range():
    from paper_2303_02317_b200.workloads import draw_config

    a, b = draw_config(3, n=64), draw_config(3, n=64)
    assert np.array_equal(a.S, b.S) and np.array_equal(a.E, b.E)
    assert np.all((a.S >= 50) & (a.S <= 150)) and np.all(a.Y == 0.0) and np.all(a.T == 2 ** 14)
    assert np.all((a.R >= 0.01) & (a.R <= 0.08)) and np.all((a.V >= 0.1) & (a.V <= 0.6))
    c1 = draw_config(1, n=32)
    assert np.all(c1.kind == 0) and np.all(c1.T == 4096)
    c2 = draw_config(2, n=32)
    assert np.all((c2.Y >= 0.01) & (c2.Y <= 0.06))
    h = draw_config(6, n=8)
    assert np.all(h.T == 2 ** 16) and np.all(h.kind == 2)
    # every drawn option is accepted by the discretisation (rejected draws are redrawn)
    status, _, _, _ = __import__("paper_2303_02317_b200._native", fromlist=["inspect"]).inspect(
        a.kind, a.S, a.K, a.R, a.Y, a.V, a.E, a.T)
    assert np.all(status == 0)


def test_c5_composition():
    from paper_2303_02317_b200.workloads import draw_config

    b = draw_config(5, n=3000)
    assert np.sum(b.kind == 0) == 1000 and np.sum(b.kind == 1) == 1000 and np.sum(b.kind == 2) == 1000
    assert set(np.unique(b.T).tolist()) <= {2 ** e for e in range(10, 17)}


def test_lpt_shards_partition_and_balance():
    from paper_2303_02317_b200.shard import lpt_shards, option_cost
    from paper_2303_02317_b200.workloads import draw_config

    b = draw_config(5, n=3000)
    for world in (1, 2, 4, 8):
        sh = lpt_shards(b.kind, b.T, world)
        allidx = np.sort(np.concatenate(sh))
        assert np.array_equal(allidx, np.arange(len(b)))
        loads = [option_cost(b.kind[s], b.T[s]).sum() for s in sh]
        assert max(loads) <= 1.02 * (sum(loads) / world) + option_cost(2, 2 ** 16)


def test_api_argument_checks_before_device():
    import paper_2303_02317_b200 as fl

    k = fl.Kernel(np.array([0.5, 0.5]), 0)
    assert np.array_equal(fl.kernel_power(k, 0).weights, [1.0])
    assert np.array_equal(fl.kernel_power(k, 1).weights, [0.5, 0.5])
    with pytest.raises(fl.ValidationError):
        fl.kernel_power(k, -1)
    with pytest.raises(fl.InsufficientWidthError):
        fl.apply_linear_steps(fl.GridRow(0, 0, np.ones(3)), k, 5)
    with pytest.raises(fl.NumericalIntegrityError):  # non-finite weights never reach the device
        fl.kernel_power(fl.Kernel(np.array([0.2, np.inf, 0.2, 0.2]), 0), 3)
    assert np.array_equal(fl.kernel_power(fl.Kernel(np.zeros(3), -1), 4).weights, np.zeros(9))  # all-zero kernel
    with pytest.raises(fl.ValidationError):
        fl.Kernel(np.array([]), 0)
    spec = fl.OptionSpec(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024)
    with pytest.raises(fl.ValidationError):
        fl.fft_forward(np.ones(3))
    with pytest.raises(fl.ValidationError):
        fl.fft_inverse(np.ones((2, 2)))
    with pytest.raises(fl.ValidationError):
        fl.convolve(np.ones(0), np.ones(2))
    disc = fl.discretize_bsm(spec)
    st = fl.initial_row(disc)
    assert st.boundary == 0 and st.segment.first_col == 1 and len(st.segment) == disc.k_star + 1024
    with pytest.raises(fl.GeometryError):
        fl.solve_bsm_trapezoid(disc, st, 0)
    top = fl.top_row_state(fl.OptionSpec(100.0, 90.0, 0.03, 0.07, 0.25, 365, 512))
    assert top.boundary == 251  # first exercise column of the terminal row is 252 (test_american.py)
    assert math.isclose(fl.bsm_green_value(disc, 0), 0.0)


def test_model_frozen_constants():
    import paper_2303_02317_b200 as fl

    d = fl.discretize_bsm(fl.OptionSpec(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024), 0.4)
    assert (d.omega, d.d_tau, d.d_s, d.k_star) == (2.4999999999999996, 1.9531250000000004e-05,
                                                  0.0069877124296868435, 0)
    assert (d.coef_down, d.coef_mid, d.coef_up) == (0.39790368627109396, 0.199951171875, 0.4020963137289061)


def test_native_shard_plan_matches_python_lpt():
    """fl_shard_plan (C++, behind fl_price_batch_multi) == shard.lpt_shards."""
    from paper_2303_02317_b200._native import shard_plan
    from paper_2303_02317_b200.shard import lpt_shards
    from paper_2303_02317_b200.workloads import draw_config

    b = draw_config(5, n=3000)
    for k in (1, 2, 3, 4, 8):
        owner = shard_plan(b.kind, b.T, k)
        for r, idx in enumerate(lpt_shards(b.kind, b.T, k)):
            assert np.array_equal(np.nonzero(owner == r)[0], idx), (k, r)


def test_oracle_margins_match_reference_goldens():
    """The oracle's boundary margins (tie evidence for boundary parity) are
    bit-identical to the reference's own, recorded in the goldens."""
    from conftest import golden
    from oracle import port

    for name in ("c3_fast", "c2_fast", "small_fast"):
        g = golden(name)
        for i in range(0, g.n, max(1, g.n // 12)):
            if str(g.err_kind[i]) or g.kind[i] == 0:
                continue
            fn = port.put_fast if g.kind[i] == 2 else port.call_fast
            _, t, c, m = fn(*g.args(i), margins=True)
            tr, cr = g.boundary(i)
            assert np.array_equal(t, tr) and np.array_equal(c, cr)
            assert np.array_equal(m, g.margins(i), equal_nan=True), (name, i)


def test_boundary_check_rules():
    """conftest.boundary_check: equal records pass; a shift passes only over
    cells the reference certifies as ties; later records are then free."""
    from conftest import NMARG, boundary_check

    t = np.array([0, 10, 20])
    c = np.array([0, -5, -9])
    marg = np.full((3, NMARG), 1e-3)
    assert boundary_check(2, 100.0, t, c, t, c, marg)[0]
    # put: device boundary one column right (cell -4 exercise on device) -> needs margin at d=+1
    c2 = np.array([0, -4, -7])
    assert not boundary_check(2, 100.0, t, c2, t, c, marg)[0]
    marg[1, NMARG // 2 + 1] = 5e-10
    ok, nt, _ = boundary_check(2, 100.0, t, c2, t, c, marg)
    assert ok and nt == 1
    # a shift of two needs both cells
    c3 = np.array([0, -3, -9])
    assert not boundary_check(2, 100.0, t, c3, t, c, marg)[0]
    # no margin evidence (NaN) -> no slack
    marg[1, :] = np.nan
    assert not boundary_check(2, 100.0, t, c2, t, c, marg)[0]
    # differing record times fail
    assert not boundary_check(2, 100.0, np.array([0, 11, 20]), c, t, c, np.full((3, NMARG), 0.0))[0]
    # call: margins in currency, tolerance 1e-9 K
    mc = np.full((3, NMARG), 1e-3)
    mc[1, NMARG // 2] = 5e-8  # |lin - green| at the reference's last continuation column
    cc = np.array([5, 7, 9])
    assert boundary_check(1, 100.0, t, np.array([5, 6, 9]), t, cc, mc)[0]
    assert not boundary_check(1, 1.0, t, np.array([5, 6, 9]), t, cc, mc)[0]
