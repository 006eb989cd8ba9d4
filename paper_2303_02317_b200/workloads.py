"""Seeded synthetic option batches for the BASELINE.json configs.

The reference measures on no public dataset; these generators stand in for
the configs named in ``BASELINE.json`` (C1..C5) with the documented ranges
(SURVEY.md 8(d)).  Draw order per option: S, K, R, Y, V, E (Y skipped for
puts, fixed at 0); C5 draws the exponent of T after the option's parameters
and assigns types in contiguous blocks.  Draws the reference rejects with
StabilityError / DomainError / ValidationError are redrawn, as the
reference's own tests do (test_bsm.py:50-67).

The generator is host logic shared by tests, bench and goldens; it never
prices anything.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .model import OptionSpec, PricingError, derive_binomial_params

__all__ = ["KIND_EURO", "KIND_CALL", "KIND_PUT", "Batch", "draw_config", "CONFIG_INFO"]

KIND_EURO, KIND_CALL, KIND_PUT = 0, 1, 2
SEED = 20261019

_EURO_RANGES = dict(S=(50.0, 150.0), K=(50.0, 150.0), R=(0.01, 0.05),
                    Y=(0.0, 0.03), V=(0.1, 0.5), E=(30.0, 365.0))
_CALL_RANGES = dict(_EURO_RANGES, Y=(0.01, 0.06))
_PUT_RANGES = dict(S=(50.0, 150.0), K=(50.0, 150.0), R=(0.01, 0.08),
                   Y=None, V=(0.1, 0.6), E=(30.0, 730.0))

CONFIG_INFO = {
    1: "binomial European call, 1024 options, T=4096",
    2: "binomial American call (Y~U[.01,.06]), 256 options, T=2^14",
    3: "BSM American put (lambda=0.4), 256 options, T=2^14",
    4: "64 BSM puts + 64 American calls, T=2^18",
    5: "65536 mixed options (euro/call/put thirds), T=2^U{10..16}",
    6: "BSM American put headline: C3 distribution at T=2^16 (batch 256)",
}


@dataclass
class Batch:
    """Struct-of-arrays option batch (host, numpy)."""

    kind: np.ndarray  # int8: 0 euro, 1 American call, 2 BSM put
    S: np.ndarray
    K: np.ndarray
    R: np.ndarray
    Y: np.ndarray
    V: np.ndarray
    E: np.ndarray
    T: np.ndarray  # int64

    def __len__(self) -> int:
        return int(self.S.shape[0])

    def subset(self, idx) -> "Batch":
        idx = np.asarray(idx)
        return Batch(*(getattr(self, f)[idx] for f in
                       ("kind", "S", "K", "R", "Y", "V", "E", "T")))

    def spec(self, i: int) -> OptionSpec:
        return OptionSpec(float(self.S[i]), float(self.K[i]), float(self.R[i]),
                          float(self.Y[i]), float(self.V[i]), float(self.E[i]),
                          int(self.T[i]))


def _accept(kind: int, s: OptionSpec) -> bool:
    try:
        if kind == KIND_PUT:
            from .bsm import discretize_bsm  # local import: bsm imports native lazily

            discretize_bsm(s, 0.4)
        else:
            derive_binomial_params(s)
    except PricingError:
        return False
    return True


def _draw_one(rng, kind: int, T: int | None, exp_range=None):
    rngs = {KIND_EURO: _EURO_RANGES, KIND_CALL: _CALL_RANGES, KIND_PUT: _PUT_RANGES}[kind]
    while True:
        vals = {}
        for key in ("S", "K", "R", "Y", "V", "E"):
            lohi = rngs[key]
            if lohi is None:
                vals[key] = 0.0
                continue
            lo, hi = lohi
            vals[key] = float(rng.uniform(lo, hi))
        t = T if T is not None else int(2 ** int(rng.integers(exp_range[0], exp_range[1] + 1)))
        spec = OptionSpec(vals["S"], vals["K"], vals["R"], vals["Y"], vals["V"], vals["E"], t)
        if _accept(kind, spec):
            return spec


def _build(kinds, specs) -> Batch:
    n = len(specs)
    b = Batch(np.asarray(kinds, dtype=np.int8), *(np.empty(n) for _ in range(6)),
              np.empty(n, dtype=np.int64))
    for i, s in enumerate(specs):
        b.S[i], b.K[i], b.R[i], b.Y[i] = s.spot, s.strike, s.rate, s.dividend_yield
        b.V[i], b.E[i], b.T[i] = s.volatility, s.days_to_expiry, s.steps
    return b


def draw_config(config_id: int, n: int | None = None, T: int | None = None) -> Batch:
    """Seeded batch for config ``config_id`` (optionally resized / re-stepped).

    ``rng = default_rng([config_id, 20261019])``; n and T default to the
    BASELINE.json sizes.  Config 6 is the headline put batch (C3 ranges,
    T=2^16) with its own seed stream.
    """
    rng = np.random.default_rng([config_id, SEED])
    if config_id == 1:
        n = 1024 if n is None else n
        specs = [_draw_one(rng, KIND_EURO, T or 4096) for _ in range(n)]
        return _build([KIND_EURO] * n, specs)
    if config_id == 2:
        n = 256 if n is None else n
        specs = [_draw_one(rng, KIND_CALL, T or 2 ** 14) for _ in range(n)]
        return _build([KIND_CALL] * n, specs)
    if config_id in (3, 6):
        n = 256 if n is None else n
        t = T or (2 ** 14 if config_id == 3 else 2 ** 16)
        specs = [_draw_one(rng, KIND_PUT, t) for _ in range(n)]
        return _build([KIND_PUT] * n, specs)
    if config_id == 4:
        n = 64 if n is None else n
        t = T or 2 ** 18
        specs = [_draw_one(rng, KIND_PUT, t) for _ in range(n)]
        specs += [_draw_one(rng, KIND_CALL, t) for _ in range(n)]
        return _build([KIND_PUT] * n + [KIND_CALL] * n, specs)
    if config_id == 5:
        n = 65536 if n is None else n
        ne = n - 2 * (n // 3)
        nc = n // 3
        kinds = [KIND_EURO] * ne + [KIND_CALL] * nc + [KIND_PUT] * nc
        specs = [_draw_one(rng, k, T, (10, 16)) for k in kinds]
        return _build(kinds, specs)
    raise ValueError(f"unknown config {config_id}")
