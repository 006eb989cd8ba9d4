"""Pin the CPU oracle (oracle/port.py + oracle/loops.c) before trusting it:
against the reference's own frozen values and against the golden vectors
produced by running the reference itself (tests/golden/make_golden.py).
CPU only."""

from __future__ import annotations

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, price_close

from oracle import port  # test infrastructure: the checker

NAMES = {0: "euro", 1: "call", 2: "put"}


def _oracle(kind, args, method):
    k = NAMES[kind]
    if method == "fast":
        if k == "euro":
            return port.euro_fast(*args), None
        if k == "call":
            p, t, c = port.call_fast(*args)
            return p, (t, c)
        p, t, c = port.put_fast(*args)
        return p, (t, c)
    if k == "euro":
        return port.euro_baseline(*args), None
    if k == "call":
        p, t, c = port.call_baseline(*args)
        return p, (t, c)
    p, t, c = port.put_baseline(*args)
    return p, (t, c)


def _check_golden(name, idx=None, exact=True):
    g = golden(name)
    method = str(g.method)
    for i in (range(g.n) if idx is None else idx):
        ek = str(g.err_kind[i])
        try:
            p, bnd = _oracle(int(g.kind[i]), g.args(i), method)
        except port.OracleError as e:
            assert e.kind == ek, (name, i, e.kind, ek)
            if ek in ("ValidationError", "StabilityError"):  # the classes that carry .field / .weight
                assert e.field == str(g.err_field[i]), (name, i, e.field, g.err_field[i])
            continue
        except ValueError:  # the reference's own math-domain failure (american.py:403), mirrored
            assert ek == "ValueError", (name, i, ek)
            continue
        assert ek == "", (name, i, "oracle priced an option the reference rejects", ek)
        if exact:
            assert p == g.price[i], (name, i, p, g.price[i])
        else:
            assert price_close(p, g.price[i], g.K[i]), (name, i, p, g.price[i])
        if bnd is not None:
            t, c = g.boundary(i)
            assert np.array_equal(bnd[0], t) and np.array_equal(bnd[1], c), (name, i)


def test_reference_frozen_values():
    """The reference's own pinned literals (test_binomial.py:42-47,
    test_american.py:38-39, test_bsm.py:31-47)."""
    assert port.euro_baseline(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024) == 10.448630960582836
    assert port.call_baseline(100.0, 90.0, 0.03, 0.07, 0.25, 365, 512)[0] == 13.221948275290686
    assert port.call_baseline(150.0, 80.0, 0.09, 0.05, 0.15, 365, 512)[0] == 70.04621199751995
    assert port.put_baseline(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024)[0] == 6.090559894890663
    d = port.discretize_put(100.0, 100.0, 0.05, 0.0, 0.2, 365, 1024, 0.4)
    assert d["k_star"] == 0
    assert d["cd"] == 0.39790368627109396
    assert d["cm"] == 0.199951171875
    assert d["cu"] == 0.4020963137289061
    assert d["omega"] == 2.4999999999999996
    assert d["d_tau"] == 1.9531250000000004e-05
    assert d["d_s"] == 0.0069877124296868435
    # first exercise column of the terminal row of the American reference spec
    _, t, c = port.call_baseline(100.0, 90.0, 0.03, 0.07, 0.25, 365, 512)
    assert c[t == 512][0] == 252


def test_edge_goldens_bit_exact():
    _check_golden("edge_fast")
    _check_golden("edge_baseline")


def test_small_goldens_bit_exact():
    _check_golden("small_fast", idx=range(0, 96, 3))
    _check_golden("small_baseline", idx=range(0, 96, 6))


def test_config_goldens_sample():
    _check_golden("c1_fast", idx=range(0, 1024, 64))
    _check_golden("c2_fast", idx=range(0, 256, 64))
    _check_golden("c3_fast", idx=range(0, 256, 64))
    _check_golden("c5_fast", idx=range(0, 42, 6))


@pytest.mark.slow
def test_headline_golden_sample():
    _check_golden("c6_fast", idx=range(0, 32, 16))


def test_kernel_power_and_corr_vs_reference_ops():
    z = np.load(os.path.join(GOLDEN, "ops.npz"))
    for k in range(int(z["n_kp"])):
        w, h = z[f"kp{k}_w"], int(z[f"kp{k}_h"])
        got = port.kernel_power(w, h)
        ref = z[f"kp{k}_out"]
        assert got.shape == ref.shape
        assert np.array_equal(got, ref), k  # same pocketfft / long-double recurrence -> identical
        out = port.valid_corr(z[f"kp{k}_row"], got)
        assert np.array_equal(out, z[f"kp{k}_als"]), k


def test_trapezoid_ops_vs_reference():
    z = np.load(os.path.join(GOLDEN, "ops.npz"))
    for k in range(int(z["n_ct"])):
        S, K, R, Y, V, E, T = z[f"ct{k}_spec"]
        p = port.derive_binomial(S, K, R, Y, V, E, int(T))
        ctx = port._CallCtx(S, K, p, 256)
        jp, out = port.call_trapezoid(int(z[f"ct{k}_i"]), int(z[f"ct{k}_j"]), int(z[f"ct{k}_h"]),
                                      z[f"ct{k}_run"], ctx)
        assert jp == int(z[f"ct{k}_jp"])
        assert np.array_equal(out, z[f"ct{k}_out"])


def test_oracle_errors_mirror_reference():
    with pytest.raises(port.OracleError) as e:
        port.put_fast(100.0, 0.0, 0.05, 0.0, 0.2, 365, 64)
    assert e.value.kind == "DomainError"
    with pytest.raises(port.OracleError) as e:
        port.euro_fast(-1.0, 100.0, 0.05, 0.0, 0.2, 365, 64)
    assert e.value.kind == "ValidationError" and e.value.field == "spot"
    assert math.isfinite(port.put_fast(100.0, 100.0, 0.05, 0.0, 0.2, 365, 300)[0])
