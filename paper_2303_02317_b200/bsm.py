"""American put on the anchored log-price FD grid -- drop-in for ``fftlattice.bsm``.

Host side only: grid constants are derived here (same formula order as the
reference bsm.py:150-229); every price, boundary and row comes from the CUDA
library through :mod:`paper_2303_02317_b200._native`.  There is no CPU
fallback: without the built library these functions raise.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .model import (
    NO_GREEN,
    BoundarySeries,
    DomainError,
    GeometryError,
    GridRow,
    OptionSpec,
    StabilityError,
    UnsupportedCombinationError,
    ValidationError,
    validate_spec,
)

__all__ = [
    "DEFAULT_BSM_CUTOFF",
    "DEFAULT_LAMBDA",
    "BsmDiscretization",
    "PutRowState",
    "PutResult",
    "discretize_bsm",
    "bsm_green_value",
    "initial_row",
    "baseline_put_fd",
    "solve_bsm_trapezoid",
    "fast_put_bsm",
    "price_put_batch",
]

#: Reference recursion cutoff (bsm.py:59); governs dispatch (T <= 2*cutoff
#: -> baseline) and the apex finish (rem <= 2*cutoff).  The GPU recursion uses
#: its own, smaller, leaf height internally (results agree to rounding).
DEFAULT_BSM_CUTOFF = 128
DEFAULT_LAMBDA = 0.4  # bsm.py:66


@dataclass(frozen=True, slots=True)
class BsmDiscretization:
    """Grid constants of one put problem (bsm.py:70-106)."""

    steps: int
    omega: float
    tau_max: float
    d_tau: float
    d_s: float
    k_star: int
    lam: float
    coef_down: float
    coef_mid: float
    coef_up: float


@dataclass(frozen=True)
class PutRowState:
    """Continuation values right of the exercise boundary (bsm.py:109-131)."""

    time_index: int
    boundary: int
    segment: GridRow

    def __post_init__(self) -> None:
        if len(self.segment) == 0:
            raise GeometryError("put row state requires a nonempty segment")
        if self.segment.first_col != self.boundary + 1:
            raise GeometryError(
                "segment must start immediately above the boundary: expected "
                f"first column {self.boundary + 1}, got {self.segment.first_col}")


@dataclass(frozen=True)
class PutResult:
    """Price plus the last-exercise-column record (bsm.py:134-147)."""

    price: float
    boundaries: BoundarySeries
    rows: dict[int, GridRow] | None = field(default=None)


def discretize_bsm(spec: OptionSpec, lam: float = DEFAULT_LAMBDA,
                   steps: int | None = None) -> BsmDiscretization:
    """Anchored grid + stability checks; reference order of operations."""
    validate_spec(spec)
    n = spec.steps if steps is None else steps
    if n < 1:
        raise ValidationError("steps", "steps must be >= 1")
    if not (math.isfinite(lam) and lam > 0.0):
        raise ValidationError("lam", f"lambda must be positive, got {lam!r}")
    if spec.strike <= 0.0:
        raise DomainError("put grid requires a positive strike")
    years = spec.years
    omega = 2.0 * spec.rate / (spec.volatility ** 2)
    tau_max = 0.5 * spec.volatility ** 2 * years
    d_tau = tau_max / n
    d_s = math.sqrt(d_tau / lam)
    lm = math.log(spec.spot / spec.strike)
    k_star = round(lm / d_s)
    if abs(k_star) > 8 * n:
        raise DomainError(
            f"spot lies too many grid nodes from the strike: |{k_star}| > {8 * n}")
    if k_star != 0:
        d_s = lm / k_star
    lam_eff = d_tau / (d_s * d_s)
    drift = (omega - 1.0) * d_tau / (2.0 * d_s)
    cu = lam_eff + drift
    cd = lam_eff - drift
    cm = 1.0 - omega * d_tau - 2.0 * lam_eff
    if cm < 0.0:
        raise StabilityError(
            "coef_mid", f"centre weight {cm:.6g} is negative; choose a smaller lambda")
    if cu < 0.0:
        raise StabilityError(
            "coef_up", f"upper weight {cu:.6g} is negative; increase steps or adjust lambda")
    if cd < 0.0:
        raise StabilityError(
            "coef_down", f"lower weight {cd:.6g} is negative; increase steps or adjust lambda")
    return BsmDiscretization(n, omega, tau_max, d_tau, d_s, k_star, lam, cd, cm, cu)


def bsm_green_value(disc: BsmDiscretization, col: int) -> float:
    """Unclipped rescaled payoff 1 - e^(col d_s) (bsm.py:232-235)."""
    return 1.0 - math.exp(col * disc.d_s)


def initial_row(disc: BsmDiscretization) -> PutRowState:
    """Payoff-row state: boundary 0, zeros on cols 1..k*+T (bsm.py:247-270)."""
    width = disc.k_star + disc.steps
    if width < 1:
        raise DomainError(
            "the payoff row has no continuation cells; the spot is deep enough "
            "in the money that the price is strike - spot")
    return PutRowState(0, 0, GridRow(0, 1, np.zeros(width, dtype=np.float64)))


def baseline_put_fd(spec: OptionSpec, lam: float = DEFAULT_LAMBDA, steps: int | None = None, *,
                    record_rows: tuple[int, ...] | None = None) -> PutResult:
    """O(T^2) projected march over the shrinking window, on the device; the
    last green column of every row is recorded (bsm.py:273-338)."""
    from . import _pricing

    if record_rows is not None:
        # snapshots of the valid window of the named rows (bsm.py:296-322), on the device
        from . import _native

        disc = discretize_bsm(spec, lam, steps)
        n = disc.steps
        targets = sorted({int(t) for t in record_rows if 0 < t <= n})
        price, cols, snaps = _native.put_march_rows(disc.coef_down, disc.coef_mid, disc.coef_up, disc.d_s,
                                                    spec.strike, disc.k_star, n, targets)
        lo = disc.k_star - n
        rows = {t: GridRow(time_index=t, col_offset=lo + t, values=v) for t, v in snaps.items()}
        series = BoundarySeries(times=np.arange(n + 1, dtype=np.int64), columns=cols)
        return PutResult(price=price, boundaries=series, rows=rows)
    price, series = _pricing.price_one(_pricing.KIND_PUT, spec, method=_pricing.BASELINE, lam=float(lam),
                                       steps=steps)
    return PutResult(price=price, boundaries=series)


def fast_put_bsm(spec: OptionSpec, lam: float = DEFAULT_LAMBDA, steps: int | None = None, *,
                 base_cutoff: int = DEFAULT_BSM_CUTOFF, parallel: bool = False,
                 record_rows: bool = False) -> PutResult:
    """American put by boundary-tracking FFT recursion on the device
    (bsm.py:585-676): same dispatch (deep in the money -> K - S, T <= 2*cutoff
    -> the O(T^2) march), same stage schedule, same handoff-row record.
    ``parallel`` is accepted and has no effect on results."""
    del parallel
    from . import _pricing

    if record_rows:
        disc = discretize_bsm(spec, lam, steps)
        n = disc.steps
        if base_cutoff < 1:
            raise ValidationError("base_cutoff", "base_cutoff must be >= 1")
        if disc.k_star > -n and n > 2 * base_cutoff:  # the stage loop runs: snapshot every handoff row
            from . import _native

            price, status, times, cols, flat = _native.put_fast_rows(
                spec.spot, spec.strike, spec.rate, spec.volatility, spec.days_to_expiry, n, float(lam),
                int(base_cutoff))
            err = _native.status_error(status)
            if err is not None:
                raise err
            rows, off = {}, 0
            for t, f in zip(times[1:].tolist(), cols[1:].tolist()):
                m = disc.k_star + n - t - f
                rows[t] = GridRow(time_index=t, col_offset=f + 1, values=flat[off:off + m])
                off += m
            return PutResult(price=price, boundaries=BoundarySeries(times, cols), rows=rows)

    price, series = _pricing.price_one(_pricing.KIND_PUT, spec, method=_pricing.FAST, lam=float(lam),
                                       steps=steps, put_cutoff=int(base_cutoff))
    return PutResult(price=price, boundaries=series)


def price_put_batch(S, K, R, V, E, T, *, lam: float = DEFAULT_LAMBDA, method: str = "fast",
                    base_cutoff: int = DEFAULT_BSM_CUTOFF):
    """Batched American puts (one device call, Y = 0).  Returns (price, status)."""
    from . import _pricing

    m = _pricing.FAST if method == "fast" else _pricing.BASELINE
    S = np.asarray(S, dtype=np.float64)
    return _pricing.price_many(np.int8(_pricing.KIND_PUT), S, K, R, np.zeros_like(S), V, E, T, method=m,
                               lam=float(lam), put_cutoff=int(base_cutoff))


def solve_bsm_trapezoid(disc: BsmDiscretization, state: PutRowState, height: int, *,
                        base_cutoff: int = DEFAULT_BSM_CUTOFF, parallel: bool = False) -> PutRowState:
    """Advance a put row state ``height`` steps on the device, tracking the
    boundary (bsm.py:504-554): far jump + boundary recursion of one stage."""
    del parallel
    if height < 1:
        raise GeometryError("height must be >= 1")
    width = len(state.segment)
    if width < 2 * height:
        raise GeometryError(
            f"segment holds {width} continuation values; advancing {height} steps requires at least "
            f"{2 * height}")
    if base_cutoff < 1:
        raise ValidationError("base_cutoff", "base_cutoff must be >= 1")
    from . import _native

    kp, seg = _native.put_trapezoid(disc.coef_down, disc.coef_mid, disc.coef_up, disc.d_s, int(base_cutoff),
                                    int(state.boundary), state.segment.values, int(height))
    t = state.time_index + height
    return PutRowState(time_index=t, boundary=kp, segment=GridRow(time_index=t, col_offset=kp + 1, values=seg))
