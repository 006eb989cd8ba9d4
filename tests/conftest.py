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

    def args(self, i: int):
        return (float(self.S[i]), float(self.K[i]), float(self.R[i]), float(self.Y[i]),
                float(self.V[i]), float(self.E[i]), int(self.T[i]))


def golden(name: str) -> Golden:
    return Golden(name)


def price_close(got: float, ref: float, strike: float, rel: float = 1e-9) -> bool:
    """BASELINE.json parity rule: |d| <= 1e-9 * max(|ref|, K)."""
    return abs(got - ref) <= rel * max(abs(ref), strike)


@pytest.fixture(scope="session")
def native():
    from paper_2303_02317_b200 import _native

    return _native.lib()
