"""American call by trapezoid decomposition -- drop-in for ``fftlattice.american``.

``fast_american_call`` (american.py:428-530) keeps the reference signature,
dispatch and ``AmericanCallResult`` record (terminal row, row T-1, every
trapezoid interface, row 0); the whole solve -- junction row, trapezoid
halving recursion, strips, residual -- runs in csrc/fl_call.cu.  The row-state
value types and ``top_row_state`` (an analytic boundary search,
american.py:260-295) are host logic.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _pricing
from .binomial import AmericanCallResult
from .model import (
    BinomialParams,
    GeometryError,
    GridRow,
    OptionSpec,
    ValidationError,
    derive_binomial_params,
    green_value_binomial,
)

__all__ = [
    "DEFAULT_BASE_CUTOFF",
    "RedRowState",
    "TrapezoidProblem",
    "top_row_state",
    "solve_trapezoid",
    "fast_american_call",
    "price_american_call_batch",
]

DEFAULT_BASE_CUTOFF = 256  # american.py:53


@dataclass(frozen=True, slots=True)
class RedRowState:
    """Continuation run of one lattice row (american.py:56-82)."""

    time_index: int
    boundary: int
    segment: GridRow

    def __post_init__(self) -> None:
        if len(self.segment) and self.segment.last_col != self.boundary:
            raise GeometryError(
                f"segment ends at column {self.segment.last_col}, boundary is {self.boundary}")


@dataclass(frozen=True, slots=True)
class TrapezoidProblem:
    """One boundary-hugging trapezoid (american.py:85-113)."""

    time_index: int
    boundary: int
    height: int
    run: GridRow

    def __post_init__(self) -> None:
        if self.height < 1:
            raise GeometryError("trapezoid height must be >= 1")
        if len(self.run) == 0 or self.run.last_col != self.boundary:
            raise GeometryError("run must be nonempty and end exactly at the boundary")
        if self.height > len(self.run):
            raise GeometryError(f"height {self.height} exceeds red-run width {len(self.run)}")
        if self.height > self.time_index:
            raise GeometryError(f"height {self.height} exceeds remaining rows {self.time_index}")


def top_row_state(spec: OptionSpec, params: BinomialParams | None = None) -> RedRowState:
    """Terminal-row continuation run: analytic guess corrected by exercise
    tests so ties resolve as the baseline does (american.py:260-295)."""
    p = derive_binomial_params(spec) if params is None else params
    n = spec.steps
    if spec.strike <= 0.0:
        boundary = -1
    else:
        guess = math.floor(0.5 * n + math.log(spec.strike / spec.spot) / (2.0 * p.log_up))
        boundary = min(max(guess, -1), n)
        while boundary < n and green_value_binomial(spec, p, n, boundary + 1) <= 0.0:
            boundary += 1
        while boundary >= 0 and green_value_binomial(spec, p, n, boundary) > 0.0:
            boundary -= 1
    return RedRowState(time_index=n, boundary=boundary, segment=GridRow(n, 0, np.zeros(boundary + 1)))


def fast_american_call(spec: OptionSpec, params: BinomialParams | None = None, *,
                       base_cutoff: int = DEFAULT_BASE_CUTOFF, parallel: bool = False) -> AmericanCallResult:
    """American call in O(T log^2 T) on the device (american.py:428-530).

    ``parallel`` is accepted for signature compatibility; the device always
    runs the two halves of every recursion node concurrently and results do
    not depend on it (the reference guarantees the same)."""
    del parallel
    if int(base_cutoff) != base_cutoff or base_cutoff < 1:
        # the reference validates base_cutoff only on its recursion path; the
        # device rejects it up front with the same exception
        raise ValidationError("base_cutoff", "base_cutoff must be >= 1")
    price, series = _pricing.price_one(_pricing.KIND_CALL, spec, method=_pricing.FAST,
                                       call_cutoff=int(base_cutoff), params=params)
    return AmericanCallResult(price=price, boundaries=series)


def price_american_call_batch(S, K, R, Y, V, E, T, *, method: str = "fast",
                              base_cutoff: int = DEFAULT_BASE_CUTOFF):
    """Batched American calls (one device call).  Returns (price, status)."""
    m = _pricing.FAST if method == "fast" else _pricing.BASELINE
    return _pricing.price_many(np.int8(_pricing.KIND_CALL), S, K, R, Y, V, E, T, method=m,
                               call_cutoff=int(base_cutoff))


def solve_trapezoid(spec: OptionSpec, problem: TrapezoidProblem, params: BinomialParams | None = None, *,
                    base_cutoff: int = DEFAULT_BASE_CUTOFF, parallel: bool = False) -> RedRowState:
    """Sweep one trapezoid on the device (american.py:298-358): the left
    columns by one composed jump, the boundary strip by the halving recursion."""
    del parallel
    from . import _native

    p = derive_binomial_params(spec) if params is None else params
    if problem.boundary > problem.time_index:
        raise GeometryError(f"boundary {problem.boundary} exceeds row width {problem.time_index}")
    first = problem.run.first_col
    jp, vals = _native.call_trapezoid(spec.spot, spec.strike, p.weight_down, p.weight_up, p.log_up,
                                      int(base_cutoff), problem.time_index, problem.boundary, first,
                                      problem.run.values, problem.height)
    t = problem.time_index - problem.height
    return RedRowState(time_index=t, boundary=jp, segment=GridRow(t, first, vals))
