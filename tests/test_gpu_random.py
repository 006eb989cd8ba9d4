"""Randomised GPU-vs-oracle parity over broad parameter ranges (beyond the
BASELINE draws): extreme moneyness, near-zero and large rates / yields /
volatilities, short and long expiries, T from 2 to 6000, all three kinds and
both methods, mixed in one batch.  The oracle (oracle/port.py, pinned
bit-exact to the reference) is the checker.  Statuses must agree; prices
within 1e-9 max(|ref|, K); boundary records equal except at a tie the
oracle certifies (|lin - exercise| <= 1e-9 K at every differing cell,
conftest.boundary_check)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import NMARG, boundary_check, price_close

from oracle import port

pytestmark = pytest.mark.gpu

NAMES = {0: "euro", 1: "call", 2: "put"}


def _draw(rng, n):
    rows = []
    while len(rows) < n:
        kind = int(rng.integers(0, 3))
        S = float(np.exp(rng.uniform(np.log(5.0), np.log(500.0))))
        K = float(S * np.exp(rng.uniform(-1.5, 1.5)))
        R = float(rng.choice([0.0, 1e-4, rng.uniform(0.0, 0.15)]))
        Y = 0.0 if kind == 2 else float(rng.choice([0.0, 1e-4, rng.uniform(0.0, 0.12)]))
        V = float(rng.uniform(0.02, 1.2))
        E = float(rng.uniform(1.0, 1500.0))
        T = int(rng.choice([2, 3, 17, 255, 256, 257, 300, 513, 1000, 2048, 3001, 6000]))
        rows.append((kind, S, K, R, Y, V, E, T))
    return rows


def _oracle(kind, args, method):
    k = NAMES[kind]
    try:
        if method == 0:
            if k == "euro":
                return "", port.euro_fast(*args), None
            p, t, c, m = port.call_fast(*args, margins=True) if k == "call" else port.put_fast(*args, margins=True)
            return "", p, (t, c, m)
        if k == "euro":
            return "", port.euro_baseline(*args), None
        p, t, c = port.call_baseline(*args) if k == "call" else port.put_baseline(*args)
        return "", p, (t, c, np.full((len(t), NMARG), np.nan))
    except port.OracleError as e:
        return e.kind, None, None
    except ValueError:
        return "ValueError", None, None


@pytest.mark.parametrize("method", [0, 1])
def test_random_batch_vs_oracle(method):
    from paper_2303_02317_b200 import _native

    rng = np.random.default_rng([4242, method])
    rows = _draw(rng, 160 if method == 0 else 60)
    kind = np.array([r[0] for r in rows], dtype=np.int8)
    cols = [np.array([r[i] for r in rows]) for i in range(1, 7)]
    T = np.array([r[7] for r in rows], dtype=np.int64)
    res = _native.price_batch_full(kind, *cols, T, method=method, bnd_cap=64 if method == 0 else 6002)
    errs = {0x100: "ValidationError", 0x200: "StabilityError", 0x300: "DomainError", 0x400: "GeometryError",
            0x500: "NumericalIntegrityError", 0x600: "ValueError"}
    for i, r in enumerate(rows):
        ek, p, bnd = _oracle(r[0], r[1:], method)
        st = int(res.status[i])
        if ek:
            assert errs.get(st & 0xFF00) == ek, (i, r, ek, hex(st))
            continue
        assert st == 0, (i, r, hex(st))
        assert price_close(res.price[i], p, r[2]), (i, r, res.price[i], p)
        degenerate = r[0] == 1 and r[3] <= 1e-4 and r[4] <= 1e-4
        if bnd is not None and not degenerate:
            # (a call with R ~ Y ~ 0 has continuation == exercise value in every
            # in-the-money cell: its recorded "boundary" is rounding noise in the
            # reference itself, so only its price is compared)
            t, c = res.boundary(i)
            ok, _, why = boundary_check(r[0], r[2], t, c, bnd[0], bnd[1], bnd[2])
            assert ok, (i, r, why)
