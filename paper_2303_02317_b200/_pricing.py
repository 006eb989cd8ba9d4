"""Single-spec and batched entry into the CUDA library.

The reference pricers take one ``OptionSpec`` (duck-typed on .spot, .strike,
.rate, .dividend_yield, .volatility, .days_to_expiry, .steps) and raise the
``PricingError`` family; this module turns that calling convention into
``fl_price_batch`` calls and status codes back into the same exceptions
(reference error conventions: model.py:44-97).  Everything numeric happens on
the GPU; there is no CPU path here.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .model import BinomialParams, BoundarySeries, UnsupportedCombinationError, derive_binomial_params

KIND_EURO, KIND_CALL, KIND_PUT = _native.KIND_EURO, _native.KIND_CALL, _native.KIND_PUT
FAST, BASELINE = _native.METHOD_FAST, _native.METHOD_BASELINE


def spec_arrays(specs):
    """Struct-of-arrays view of a sequence of duck-typed specs."""
    S = np.array([float(s.spot) for s in specs], dtype=np.float64)
    K = np.array([float(s.strike) for s in specs], dtype=np.float64)
    R = np.array([float(s.rate) for s in specs], dtype=np.float64)
    Y = np.array([float(s.dividend_yield) for s in specs], dtype=np.float64)
    V = np.array([float(s.volatility) for s in specs], dtype=np.float64)
    E = np.array([float(s.days_to_expiry) for s in specs], dtype=np.float64)
    T = np.array([_steps(s.steps) for s in specs], dtype=np.int64)
    return S, K, R, Y, V, E, T


def _steps(t) -> int:
    # non-integral / non-positive steps must still raise ValidationError('steps'):
    # the device validates T >= 1, a fractional value is mapped to 0 (invalid)
    try:
        ti = int(t)
    except (TypeError, ValueError, OverflowError):
        return 0
    return ti if ti == t else 0


def check_params(spec, params: BinomialParams | None) -> None:
    """The normal-limit approximations derive prob_up / discount on the
    device from the spec; caller-supplied constants must agree there (the
    lattice pricers take them: ``bparams``)."""
    if params is None:
        return
    if params != derive_binomial_params(spec):
        raise UnsupportedCombinationError(
            "the GPU normal-limit approximations derive prob_up and the discount from the spec; "
            "custom BinomialParams are supported by the lattice pricers only")


def bparams(params: BinomialParams | None):
    """Caller-supplied lattice constants as the C ABI's override row (the
    reference pricers' ``params=``, binomial.py:80/161, american.py:428)."""
    if params is None:
        return None
    return np.array([[float(params.weight_down), float(params.weight_up), float(params.log_up),
                      float(params.step_years)]])


def price_one(kind: int, spec, *, method: int = FAST, lam: float = 0.4, steps: int | None = None,
              call_cutoff: int = 256, put_cutoff: int = 128, record: bool = True,
              params: BinomialParams | None = None):
    """Price one spec on the device; returns (price, BoundarySeries | None).

    Raises the reference exception for a nonzero status."""
    S, K, R, Y, V, E, T = spec_arrays([spec])
    if steps is not None:
        T[0] = _steps(steps)
    bp = bparams(params)
    if record:
        cap = int(T[0]) + 2 if method == BASELINE else 64
        res = _native.price_batch_full(np.int8(kind), S, K, R, Y, V, E, T, lam=lam, call_cutoff=call_cutoff,
                                       put_cutoff=put_cutoff, method=method, bnd_cap=cap, bparams=bp)
    else:
        res = _native.price_batch(np.int8(kind), S, K, R, Y, V, E, T, lam=lam, call_cutoff=call_cutoff,
                                  put_cutoff=put_cutoff, method=method, bnd_cap=0, bparams=bp)
    err = _native.status_error(int(res.status[0]))
    if err is not None:
        raise err
    price = float(res.price[0])
    if not record:
        return price, None
    t, c = res.boundary(0)
    return price, BoundarySeries(t, c)


def price_many(kind, S, K, R, Y, V, E, T, *, method: int = FAST, lam: float = 0.4, call_cutoff: int = 256,
               put_cutoff: int = 128):
    """Batched pricing (host arrays).  Returns (price[n], status[n]); a row
    with a nonzero status has price 0 -- map it with status_error()."""
    res = _native.price_batch(kind, S, K, R, Y, V, E, T, lam=lam, call_cutoff=call_cutoff,
                              put_cutoff=put_cutoff, method=method, bnd_cap=0)
    return res.price, res.status
