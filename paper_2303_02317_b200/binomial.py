"""Binomial-lattice pricers -- drop-in for ``fftlattice.binomial``.

``fast_european`` (binomial.py:161-194), ``baseline_european`` (:80-91) and
``baseline_american_call`` (:94-130) with the reference signatures, result
types and exceptions; prices and boundary records come from the CUDA library
(csrc/fl_euro.cu, csrc/fl_call.cu).  ``leaf_row`` is the reference's host
helper (terminal-row payoffs) and stays numpy.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _pricing
from .model import (
    BinomialParams,
    BoundarySeries,
    GridRow,
    OptionSpec,
    derive_binomial_params,
)

__all__ = [
    "AmericanCallResult",
    "leaf_row",
    "baseline_european",
    "baseline_american_call",
    "fast_european",
    "gaussian_approx_european",
    "closed_form_european",
    "price_european_batch",
]


@dataclass(frozen=True, slots=True)
class AmericanCallResult:
    """Price plus first-exercise-column record (binomial.py:41-55); ``rows`` /
    ``exercise_masks`` are filled by ``baseline_american_call(keep_grid=True)``."""

    price: float
    boundaries: BoundarySeries
    rows: list[np.ndarray] | None = None
    exercise_masks: list[np.ndarray] | None = None


def leaf_row(spec: OptionSpec, params: BinomialParams | None = None) -> GridRow:
    """Terminal-row call values max(S u^(2j-T) - K, 0) (binomial.py:64-77)."""
    p = derive_binomial_params(spec) if params is None else params
    n = spec.steps
    j = np.arange(n + 1, dtype=np.float64)
    return GridRow(n, 0, np.maximum(spec.spot * np.exp((2.0 * j - n) * p.log_up) - spec.strike, 0.0))


def baseline_european(spec: OptionSpec, params: BinomialParams | None = None) -> float:
    """O(T^2) backward induction on the device (binomial.py:80-91)."""
    price, _ = _pricing.price_one(_pricing.KIND_EURO, spec, method=_pricing.BASELINE, record=False, params=params)
    return price


def fast_european(spec: OptionSpec, params: BinomialParams | None = None) -> float:
    """Gauged composed-kernel inner product on the device (binomial.py:161-194)."""
    price, _ = _pricing.price_one(_pricing.KIND_EURO, spec, method=_pricing.FAST, record=False, params=params)
    return price


def baseline_american_call(spec: OptionSpec, params: BinomialParams | None = None, *,
                           keep_grid: bool = False) -> AmericanCallResult:
    """O(T^2) projected induction on the device, first green per row recorded
    (binomial.py:94-130)."""
    if keep_grid:
        # every row and exercise mask retained (binomial.py:133-158), computed on the device
        from . import _native

        p = derive_binomial_params(spec) if params is None else params
        price, rows, masks, cols = _native.call_grid(spec.spot, spec.strike, p.weight_down, p.weight_up,
                                                     p.log_up, spec.steps)
        series = BoundarySeries(np.arange(spec.steps + 1, dtype=np.int64), cols)
        return AmericanCallResult(price=price, boundaries=series, rows=rows, exercise_masks=masks)
    price, series = _pricing.price_one(_pricing.KIND_CALL, spec, method=_pricing.BASELINE, params=params)
    return AmericanCallResult(price=price, boundaries=series)


def price_european_batch(S, K, R, Y, V, E, T, *, method: str = "fast"):
    """Batched European calls (one device call).  Returns (price, status)."""
    m = _pricing.FAST if method == "fast" else _pricing.BASELINE
    return _pricing.price_many(np.int8(_pricing.KIND_EURO), S, K, R, Y, V, E, T, method=m)


def _euro_approx(spec: OptionSpec, params: BinomialParams | None, method: int) -> float:
    from . import _native

    _pricing.check_params(spec, params)
    S, K, R, Y, V, E, T = _pricing.spec_arrays([spec])
    price, status = _native.euro_approx(S, K, R, Y, V, E, T, method)
    err = _native.status_error(int(status[0]))
    if err is not None:
        raise err
    return float(price[0])


def gaussian_approx_european(spec: OptionSpec, params: BinomialParams | None = None) -> float:
    """European call with the composed weights replaced by their normal limit,
    summed over a six-sigma window on the device (binomial.py:197-240)."""
    from . import _native

    return _euro_approx(spec, params, _native.METHOD_GAUSS)


def closed_form_european(spec: OptionSpec, params: BinomialParams | None = None) -> float:
    """Closed form of the normal-limit price, on the device (binomial.py:243-296)."""
    from . import _native

    return _euro_approx(spec, params, _native.METHOD_CLOSED)
