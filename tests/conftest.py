"""Shared test helpers.  ``-m gpu`` tests need a B200 and the built library;
everything else runs on CPU (oracle vs goldens, host logic, ABI symbols)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

KIND_NAMES = {0: "euro", 1: "call", 2: "put"}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


class Golden:
    """One golden fixture (tests/golden/*.npz written by make_golden.py)."""

    def __init__(self, name: str):
        z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
        self.name = name
        for k in z.files:
            setattr(self, k, z[k])
        self.n = int(self.S.shape[0])

    def boundary(self, i: int):
        a, b = int(self.bnd_off[i]), int(self.bnd_off[i + 1])
        return self.bnd_times[a:b], self.bnd_cols[a:b]

    def margins(self, i: int):
        a, b = int(self.bnd_off[i]), int(self.bnd_off[i + 1])
        return self.bnd_marg[a:b]

    def args(self, i: int):
        return (float(self.S[i]), float(self.K[i]), float(self.R[i]), float(self.Y[i]),
                float(self.V[i]), float(self.E[i]), int(self.T[i]))


def golden(name: str) -> Golden:
    return Golden(name)


NMARG = 7  # boundary margins per record: cells b-3 .. b+3 (make_golden.py)
NO_GREEN = int(np.iinfo(np.int64).min)


def boundary_check(kind: int, strike: float, tg, cg, tr, cr, marg, tol: float = 1e-9):
    """Boundary parity with tie slack tied to the reference's own margins.

    ``tg/cg`` device record times / columns, ``tr/cr`` the reference's,
    ``marg`` (n_rec x NMARG) the reference's lin - exercise at cells b-3..b+3
    around its boundary b on each record's row (put: b = the record's column,
    the last exercise column, margins in units of K; call: b = column - 1,
    the last continuation column, margins in currency).

    Records are compared in order.  The first record whose column differs
    must be a tie: every cell between the two boundaries must have
    |lin - exercise| <= tol*K in the reference (put) / <= tol*K (call), as
    north_star allows.  After a tie the two solvers may legitimately take
    different stage / trapezoid heights (they depend on the boundary), so
    later records are not compared; the price still is.  Returns
    ``(ok, n_ties, why)``.
    """
    n = min(len(tg), len(tr))
    for r in range(n):
        if tg[r] != tr[r]:
            return False, 0, f"record {r}: time {tg[r]} != {tr[r]}"
        if cg[r] == cr[r]:
            continue
        if NO_GREEN in (int(cg[r]), int(cr[r])):
            return False, 0, f"record {r} (t={tr[r]}): NO_GREEN vs column"
        shift = 0 if kind == 2 else 1
        bg, br = int(cg[r]) - shift, int(cr[r]) - shift
        lo, hi = min(bg, br) + 1, max(bg, br)
        scale = 1.0 if kind == 2 else strike
        for c in range(lo, hi + 1):
            d = c - br + NMARG // 2
            if not (0 <= d < NMARG) or not np.isfinite(marg[r, d]):
                return False, 0, f"record {r} (t={tr[r]}): column {cg[r]} vs {cr[r]}, no tie evidence"
            if abs(marg[r, d]) > tol * scale:
                return False, 0, (f"record {r} (t={tr[r]}): column {cg[r]} vs {cr[r]}, "
                                  f"margin {marg[r, d]:.3e} at column {c} is not a tie")
        return True, 1, ""
    if len(tg) != len(tr):
        return False, 0, f"{len(tg)} records vs {len(tr)}"
    return True, 0, ""


def price_close(got: float, ref: float, strike: float, rel: float = 1e-9) -> bool:
    """BASELINE.json parity rule: |d| <= 1e-9 * max(|ref|, K)."""
    return abs(got - ref) <= rel * max(abs(ref), strike)


@pytest.fixture(scope="session")
def native():
    from paper_2303_02317_b200 import _native

    return _native.lib()
