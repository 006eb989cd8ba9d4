"""CPU oracle -- TEST INFRASTRUCTURE ONLY, never the product path.

A restatement of the reference `fftlattice` pricing algorithms (numpy for the
vector work, ``oracle/loops.c`` for the five explicit inner loops) used as the
parity checker for the CUDA path.  Every function cites the reference
file:line it follows (paths relative to ``/root/reference/pkg/src/fftlattice``).

Pinning: ``tests/test_oracle_golden.py`` checks this port against the
reference's own frozen values (test_binomial.py:42-47, test_american.py:38-39,
test_bsm.py:32-47) and against golden vectors produced by importing the
reference itself (``tests/golden/make_golden.py``); in this container the port
reproduces the reference bit for bit (same numpy pocketfft, same x87 long
double, same libm, unfused loops).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline /
``--impl reference``) may import this module.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

__all__ = [
    "OracleError",
    "NONE_SEEN",
    "NO_GREEN",
    "load_loops",
    "derive_binomial",
    "discretize_put",
    "two_tap_power",
    "kernel_power",
    "valid_corr",
    "euro_fast",
    "euro_baseline",
    "call_baseline",
    "call_fast",
    "put_baseline",
    "put_fast",
    "price",
]

NONE_SEEN = -(1 << 60)  # _accel.py:46
# Boundary margins (tie evidence).  north_star lets a device boundary index
# differ from the reference's only at a tie within tolerance.  With
# ``margins=True`` the fast pricers also return, per boundary record produced
# by a leaf strip, lin - exercise on that record's row at the NMARG cells
# b-3 .. b+3 around the oracle's boundary b (b = last exercise column for the
# put, last continuation column for the call), in the reference's own
# expression order; NaN where a record is not a strip result.  Put margins
# are in units of K, call margins in currency.  Same definition as the
# golden fixtures' ``bnd_marg`` (tests/golden/make_golden.py).
NMARG = 7
_NOMARG = np.full(NMARG, np.nan)
NO_GREEN = int(np.iinfo(np.int64).min)  # model.py:41
DAYS = 365.0  # model.py:37

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class OracleError(Exception):
    """Mirror of the reference exception hierarchy (model.py:44-97).

    ``kind`` is the reference class name; ``field`` the offending field or
    weight name (``None`` where the reference carries none).
    """

    def __init__(self, kind: str, field: str | None, message: str = "") -> None:
        super().__init__(message or f"{kind}({field})")
        self.kind = kind
        self.field = field


# ---------------------------------------------------------------------------
# C loops


def load_loops():
    """Load (building on first use) ``oracle/liboracle_loops.so``."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.path.join(_HERE, "liboracle_loops.so")
    src = os.path.join(_HERE, "loops.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    lib = ctypes.CDLL(path)
    d, i64, p = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p
    lib.orc_european_backward.argtypes = [p, i64, d, d]
    lib.orc_european_backward.restype = d
    lib.orc_american_call_backward.argtypes = [p, i64, p, p, d, d, d, d, d]
    lib.orc_american_call_backward.restype = d
    lib.orc_binomial_strip_sweep.argtypes = [p, p, i64, i64, i64, i64, d, d, d, d, d]
    lib.orc_binomial_strip_sweep.restype = i64
    lib.orc_put_march_window.argtypes = [p, i64, p, i64, i64, d, d, d, p]
    lib.orc_put_march_window.restype = d
    lib.orc_bsm_strip_sweep.argtypes = [p, i64, p, i64, i64, d, d, d]
    lib.orc_bsm_strip_sweep.restype = i64
    _LIB = lib
    return lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags.c_contiguous
    return a.ctypes.data


# ---------------------------------------------------------------------------
# parameters


def _validate(S, K, R, Y, V, E, T) -> None:
    """model.py:145-175 (first violated field wins)."""
    checks = (
        ("spot", S > 0.0 and math.isfinite(S)),
        ("strike", K >= 0.0 and math.isfinite(K)),
        ("rate", R >= 0.0 and math.isfinite(R)),
        ("dividend_yield", Y >= 0.0 and math.isfinite(Y)),
        ("volatility", V > 0.0 and math.isfinite(V)),
        ("days_to_expiry", E > 0.0 and math.isfinite(E)),
        ("steps", int(T) == T and T >= 1),
    )
    for name, ok in checks:
        if not ok:
            raise OracleError("ValidationError", name)


def derive_binomial(S, K, R, Y, V, E, T) -> dict:
    """model.py:211-248, same operation order."""
    _validate(S, K, R, Y, V, E, T)
    dt = E / (DAYS * T)
    lu = V * math.sqrt(dt)
    up = math.exp(lu)
    down = 1.0 / up
    growth = math.exp((R - Y) * dt)
    p = (growth - down) / (up - down)
    if not 0.0 < p < 1.0:
        raise OracleError("ValidationError", "prob_up")
    disc = math.exp(-R * dt)
    return dict(dt=dt, up=up, down=down, p=p, disc=disc,
                wd=disc * (1.0 - p), wu=disc * p, lu=lu)


def discretize_put(S, K, R, Y, V, E, T, lam=0.4) -> dict:
    """bsm.py:150-229 (anchored log-price grid, stability checks)."""
    _validate(S, K, R, Y, V, E, T)
    n = int(T)
    if not (math.isfinite(lam) and lam > 0.0):
        raise OracleError("ValidationError", "lam")
    if K <= 0.0:
        raise OracleError("DomainError", "strike")
    years = E / DAYS
    omega = 2.0 * R / (V ** 2)
    tau_max = 0.5 * V ** 2 * years
    d_tau = tau_max / n
    d_s = math.sqrt(d_tau / lam)
    lm = math.log(S / K)
    k_star = round(lm / d_s)
    if abs(k_star) > 8 * n:
        raise OracleError("DomainError", "grid_nodes")
    if k_star != 0:
        d_s = lm / k_star
    lam_eff = d_tau / (d_s * d_s)
    drift = (omega - 1.0) * d_tau / (2.0 * d_s)
    cu = lam_eff + drift
    cd = lam_eff - drift
    cm = 1.0 - omega * d_tau - 2.0 * lam_eff
    if cm < 0.0:
        raise OracleError("StabilityError", "coef_mid")
    if cu < 0.0:
        raise OracleError("StabilityError", "coef_up")
    if cd < 0.0:
        raise OracleError("StabilityError", "coef_down")
    return dict(n=n, omega=omega, tau_max=tau_max, d_tau=d_tau, d_s=d_s,
                k_star=k_star, cd=cd, cm=cm, cu=cu)


# ---------------------------------------------------------------------------
# composed stencils and valid correlation (fft.py)


def _next_pow2(n: int) -> int:
    """fft.py:126-127."""
    return 1 << max(0, (n - 1).bit_length())


def two_tap_power(a: float, b: float, h: int) -> np.ndarray:
    """fft.py:166-200: C(h,r) a^(h-r) b^r through a long-double log cumsum."""
    if a == 0.0 or b == 0.0:
        out = np.zeros(h + 1)
        if b == 0.0:
            out[0] = a ** h
        else:
            out[h] = b ** h
        return out
    L = np.longdouble
    r = np.arange(1, h + 1, dtype=L)
    steps = np.log(abs(L(b) / L(a)) * (L(h) - r + 1.0) / r)
    lw = np.empty(h + 1, dtype=L)
    lw[0] = L(h) * np.log(abs(L(a)))
    np.cumsum(steps, out=lw[1:])
    lw[1:] += lw[0]
    out = np.exp(lw.astype(np.float64))
    if a < 0.0 or b < 0.0:
        sa = -1.0 if a < 0.0 else 1.0
        sb = -1.0 if b < 0.0 else 1.0
        idx = np.arange(h + 1)
        out *= np.where((h - idx) % 2 == 1, sa, 1.0)
        out *= np.where(idx % 2 == 1, sb, 1.0)
    return out


def kernel_power(weights: np.ndarray, h: int) -> np.ndarray:
    """fft.py:203-260: weights of h composed applications of a stencil."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    if h == 0:
        return np.array([1.0])
    if h == 1:
        return w.copy()
    if len(w) == 2:
        return two_tap_power(float(w[0]), float(w[1]), h)
    m = h * (len(w) - 1) + 1
    n = _next_pow2(m)
    pad = np.zeros(n)
    pad[: len(w)] = w
    out = np.fft.irfft(np.fft.rfft(pad) ** h, n)[:m]
    if not np.all(np.isfinite(out)):
        raise OracleError("NumericalIntegrityError", None)
    return np.ascontiguousarray(out)


def _conv_real(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """fft.py:130-158 (real path): rfft . rfft -> irfft at next_pow2(L+M-1)."""
    m = x.shape[0] + y.shape[0] - 1
    n = _next_pow2(m)
    fx = np.zeros(n)
    fy = np.zeros(n)
    fx[: x.shape[0]] = x
    fy[: y.shape[0]] = y
    return np.ascontiguousarray(np.fft.irfft(np.fft.rfft(fx) * np.fft.rfft(fy), n)[:m])


def valid_corr(vals: np.ndarray, composed: np.ndarray) -> np.ndarray:
    """american.py:180-184 / bsm.py:384-387: out[k] = sum_r W[r] vals[k+r]."""
    lw = composed.shape[0]
    full = _conv_real(vals, composed[::-1])
    return np.ascontiguousarray(full[lw - 1: vals.shape[0]])


class _Powers:
    """Per-solve composed-kernel cache (american.py:152-157, bsm.py:364-369)."""

    def __init__(self, weights):
        self.w = np.asarray(weights, dtype=np.float64)
        self.cache = {}

    def __call__(self, h):
        got = self.cache.get(h)
        if got is None:
            got = kernel_power(self.w, h)
            self.cache[h] = got
        return got


# ---------------------------------------------------------------------------
# European call (binomial.py)


def _leaf(S, K, p, n) -> np.ndarray:
    """binomial.py:64-77."""
    j = np.arange(n + 1, dtype=np.float64)
    return np.maximum(S * np.exp((2.0 * j - n) * p["lu"]) - K, 0.0)


def euro_baseline(S, K, R, Y, V, E, T) -> float:
    """binomial.py:80-91 via the O(T^2) loop (_accel.py:49-59)."""
    p = derive_binomial(S, K, R, Y, V, E, T)
    v = _leaf(S, K, p, int(T)).copy()
    return float(load_loops().orc_european_backward(_ptr(v), v.shape[0], p["wd"], p["wu"]))


def euro_fast(S, K, R, Y, V, E, T, p=None) -> float:
    """binomial.py:161-194: gauged composed weights . rescaled leaf."""
    p = derive_binomial(S, K, R, Y, V, E, T) if p is None else p
    n = int(T)
    w = kernel_power(np.array([p["wd"], p["wu"] * math.exp(2.0 * p["lu"])]), n)
    r = np.arange(n + 1, dtype=np.float64)
    leaf = np.maximum(S * math.exp(-n * p["lu"]) - K * np.exp(-2.0 * r * p["lu"]), 0.0)
    return float(np.dot(w, leaf))


# ---------------------------------------------------------------------------
# American call (binomial.py:94-130, american.py)


def call_baseline(S, K, R, Y, V, E, T, p=None):
    """binomial.py:94-130: O(T^2) projected induction; (price, times, cols)."""
    p = derive_binomial(S, K, R, Y, V, E, T) if p is None else p
    n = int(T)
    v = _leaf(S, K, p, n).copy()
    u2 = np.exp((2.0 * np.arange(n + 1, dtype=np.float64) - n) * p["lu"])
    fg = np.empty(n + 1, dtype=np.int64)
    price = float(load_loops().orc_american_call_backward(
        _ptr(v), v.shape[0], _ptr(u2), _ptr(fg), S, K, p["wd"], p["wu"], p["lu"]))
    cols = np.where(fg == NONE_SEEN, NO_GREEN, fg)
    return price, np.arange(n + 1, dtype=np.int64), cols


def _green_call(S, K, p, i, j) -> float:
    """model.py:251-262."""
    return S * math.exp((2 * j - i) * p["lu"]) - K


def _call_top_boundary(S, K, p, n) -> int:
    """american.py:260-295: last out-of-the-money terminal column."""
    if K <= 0.0:
        return -1
    b = math.floor(0.5 * n + math.log(K / S) / (2.0 * p["lu"]))
    b = min(max(b, -1), n)
    while b < n and _green_call(S, K, p, n, b + 1) <= 0.0:
        b += 1
    while b >= 0 and _green_call(S, K, p, n, b) > 0.0:
        b -= 1
    return b


def _first_green(i, j):
    """american.py:361-363."""
    return NO_GREEN if j >= i else j + 1


class _CallCtx:
    """american.py:116-165."""

    def __init__(self, S, K, p, cutoff):
        self.S, self.K, self.p, self.cutoff = S, K, p, cutoff
        self.power = _Powers([p["wd"], p["wu"]])
        self.e2 = np.exp(2.0 * np.arange(cutoff + 2, dtype=np.float64) * p["lu"])

    def e2_min(self, m):
        if self.e2.shape[0] < m:
            self.e2 = np.exp(2.0 * np.arange(m, dtype=np.float64) * self.p["lu"])
        return self.e2

    want_marg = False
    marg_last = None

    def strip(self, buf, lo, top_row, boundary, height, e2_len):
        p = self.p
        e2 = self.e2_min(e2_len)
        buf0 = buf.copy() if self.want_marg else None
        jr = int(load_loops().orc_binomial_strip_sweep(
            _ptr(buf), _ptr(e2), lo, top_row, boundary, height,
            self.S, self.K, p["wd"], p["wu"], p["lu"]))
        if buf0 is not None:
            self.marg_last = self._margins(buf0, e2, lo, top_row, boundary, height, jr)
        return jr

    def _margins(self, buf, e2, lo, top_row, boundary, height, jr):
        """lin - exercise of the strip's last row at cells jr-3 .. jr+3
        (_accel.py:143-153 expression order); see ``boundary_margins``."""
        p = self.p
        j1 = boundary
        if height > 1:
            j1 = int(load_loops().orc_binomial_strip_sweep(
                _ptr(buf), _ptr(e2), lo, top_row, boundary, height - 1,
                self.S, self.K, p["wd"], p["wu"], p["lu"]))
        m = np.full(NMARG, np.nan)
        parent = top_row - (height - 1)
        child = parent - 1
        if j1 >= lo:
            top = j1 if j1 < child else child
            bc = self.S * math.exp((2 * lo - child) * p["lu"])
            bp = self.S * math.exp((2 * lo - parent) * p["lu"])
            for d in range(-(NMARG // 2), NMARG // 2 + 1):
                c = jr + d
                if lo <= c <= top:
                    vr = buf[c + 1 - lo] if c + 1 <= j1 else bp * e2[c + 1 - lo] - self.K
                    m[d + NMARG // 2] = (p["wd"] * buf[c - lo] + p["wu"] * vr) - (bc * e2[c - lo] - self.K)
        return m


def _call_solve(i, j, h, vals, ctx):
    """american.py:201-257: halving recursion over a boundary trapezoid."""
    if h <= ctx.cutoff:
        buf = vals.copy()
        jp = ctx.strip(buf, j - h + 1, i, j, h, h + 1)
        return jp, buf[: jp - (j - h + 1) + 1]
    h1 = (h + 1) // 2
    h2 = h - h1
    mid = valid_corr(vals, ctx.power(h1))
    jm, upper = _call_solve(i, j, h1, vals[h - h1:], ctx)
    if jm < j - h1 or jm > j:
        raise OracleError("GeometryError", None)
    if mid.shape[0] != h2 or upper.shape[0] != jm - (j - h1):
        raise OracleError("GeometryError", None)
    asm = np.concatenate((mid, upper))
    blen = asm.shape[0] - h2
    bottom = valid_corr(asm, ctx.power(h2)) if blen > 0 else asm[:0]
    jp, lower = _call_solve(i - h1, jm, h2, asm[-h2:], ctx)
    if jp < jm - h2 or jp > jm:
        raise OracleError("GeometryError", None)
    if bottom.shape[0] != blen or lower.shape[0] != jp - (jm - h2):
        raise OracleError("GeometryError", None)
    return jp, np.concatenate((bottom, lower))


def call_trapezoid(i, j, h, run, ctx):
    """american.py:334-358: one trapezoid (left jump + boundary recursion)."""
    width = run.shape[0]
    strip = run[width - h:]
    left = valid_corr(run, ctx.power(h)) if width > h else run[:0]
    jp, sout = _call_solve(i, j, h, strip, ctx)
    out = np.concatenate((left, sout))
    if out.shape[0] != jp + 1 - (j + 1 - width):
        raise OracleError("GeometryError", None)
    return jp, out


def _call_junction(S, K, R, Y, p, n, top_b):
    """american.py:366-425: explicit row T-1."""
    i = n - 1
    wd, wu = p["wd"], p["wu"]

    def red(j):
        vd = _green_call(S, K, p, n, j)
        vu = _green_call(S, K, p, n, j + 1)
        lin = wd * (vd if vd > 0.0 else 0.0) + wu * (vu if vu > 0.0 else 0.0)
        return lin >= _green_call(S, K, p, i, j)

    rdt = R * p["dt"]
    ydt = Y * p["dt"]
    guess = top_b
    if rdt > 0.0 and ydt > 0.0:
        shift = math.log(K / S) + math.log(math.expm1(rdt) / math.expm1(ydt)) - (rdt - ydt)
        est = math.ceil(0.5 * i + shift / (2.0 * p["lu"])) - 1
        guess = max(guess, est)
    j = min(max(guess, -1), i)
    while j < i and red(j + 1):
        j += 1
    while j >= 0 and not red(j):
        j -= 1
    vals = np.zeros(j + 1)
    start = max(top_b, 0)
    if start <= j:
        cols = np.arange(start, j + 2, dtype=np.float64)
        leaf = S * np.exp((2.0 * cols - n) * p["lu"]) - K
        np.maximum(leaf, 0.0, out=leaf)
        vals[start:] = wd * leaf[:-1] + wu * leaf[1:]
    return i, j, vals


def call_fast(S, K, R, Y, V, E, T, base_cutoff=256, margins=False):
    """american.py:428-530: (price, times, cols), plus the per-record boundary
    margins (``boundary_margins``) when ``margins``."""
    if margins:
        return _with_margins(_call_fast, S, K, R, Y, V, E, T, base_cutoff)
    return _call_fast(S, K, R, Y, V, E, T, base_cutoff)[:3]


def _call_fast(S, K, R, Y, V, E, T, base_cutoff=256, want_marg=False):
    p = derive_binomial(S, K, R, Y, V, E, T)
    n = int(T)
    if Y == 0.0:
        price = euro_fast(S, K, R, Y, V, E, T, p)
        return price, np.array([n], dtype=np.int64), np.array(
            [_first_green(n, _call_top_boundary(S, K, p, n))], dtype=np.int64)
    if n <= base_cutoff:
        return call_baseline(S, K, R, Y, V, E, T, p)
    top_b = _call_top_boundary(S, K, p, n)
    if top_b == n:
        return (euro_fast(S, K, R, Y, V, E, T, p), np.array([n], dtype=np.int64),
                np.array([NO_GREEN], dtype=np.int64))
    times = [n]
    bounds = [_first_green(n, top_b)]
    i, j, vals = _call_junction(S, K, R, Y, p, n, top_b)
    times.append(i)
    bounds.append(_first_green(i, j))
    if j < 0:
        # american.py:478-486 returns BoundarySeries(times=[n, n-1], ...) here,
        # whose constructor rejects non-increasing times (model.py:318-328): the
        # reference raises ValidationError('times') for an all-exercise row T-1
        raise OracleError("ValidationError", "times")
    resid = math.isqrt(n - 1) + 1
    ctx = _CallCtx(S, K, p, base_cutoff)
    ctx.want_marg = want_marg
    marg = [_NOMARG, _NOMARG]
    while i > resid and j >= 0:
        h = min(j + 1, i - resid)
        ctx.marg_last = None
        j, vals = call_trapezoid(i, j, h, vals, ctx)
        i -= h
        times.append(i)
        bounds.append(_first_green(i, j))
        marg.append(_NOMARG if ctx.marg_last is None else ctx.marg_last)
    if j < 0:
        price = S - K
    else:
        buf = vals.copy()
        ctx.marg_last = None
        j0 = ctx.strip(buf, 0, i, j, i, buf.shape[0] + 1)
        price = float(buf[0]) if j0 >= 0 else S - K
        if i > 0:
            times.append(0)
            bounds.append(_first_green(0, j0))
            marg.append(_NOMARG if ctx.marg_last is None else ctx.marg_last)
    t = np.asarray(times, dtype=np.int64)
    b = np.asarray(bounds, dtype=np.int64)
    order = np.argsort(t)
    return price, t[order], b[order], np.asarray(marg)[order]


# ---------------------------------------------------------------------------
# American put (bsm.py)


def _payoff(d_s, lo, hi) -> np.ndarray:
    """bsm.py:238-244."""
    cols = np.arange(lo, hi + 1, dtype=np.float64)
    return 1.0 - np.exp(cols * d_s)


def put_baseline(S, K, R, Y, V, E, T, lam=0.4):
    """bsm.py:273-338 (no row snapshots): (price, times, cols)."""
    d = discretize_put(S, K, R, Y, V, E, T, lam)
    n = d["n"]
    lo = d["k_star"] - n
    pay = _payoff(d["d_s"], lo, d["k_star"] + n)
    v = np.maximum(pay, 0.0)
    lg = np.empty(n + 1, dtype=np.int64)
    load_loops().orc_put_march_window(_ptr(v), v.shape[0], _ptr(pay), 0, n,
                                      d["cd"], d["cm"], d["cu"], _ptr(lg))
    price = float(K * v[(v.shape[0] - 1) // 2])
    cols = np.empty(n + 1, dtype=np.int64)
    cols[0] = min(0, d["k_star"] + n)
    for r in range(1, n + 1):
        cols[r] = lo + lg[r] if lg[r] != NONE_SEEN else NO_GREEN
    return price, np.arange(n + 1, dtype=np.int64), cols


class _PutCtx:
    """bsm.py:341-369."""

    def __init__(self, d, cutoff):
        self.d, self.cutoff = d, cutoff
        self.power = _Powers([d["cd"], d["cm"], d["cu"]])

    want_marg = False
    marg_last = None

    def sweep(self, arr, pay, lo, height):
        d = self.d
        return int(load_loops().orc_bsm_strip_sweep(
            _ptr(arr), arr.shape[0], _ptr(pay), lo, height, d["cd"], d["cm"], d["cu"]))

    def margins(self, arr, pay, lo, height, kb):
        """lin - payoff of the strip's last row at cells kb-3 .. kb+3
        (_accel.py:232 expression order), units of K; see ``boundary_margins``."""
        d = self.d
        a = arr.copy()
        if height > 1:
            self.sweep(a, pay, lo, height - 1)
        hi = lo + a.shape[0] - 1
        m = np.full(NMARG, np.nan)
        for dd in range(-(NMARG // 2), NMARG // 2 + 1):
            k = kb + dd
            if lo + height <= k <= hi - height:
                lin = d["cm"] * a[k - lo] + d["cu"] * a[k + 1 - lo] + d["cd"] * a[k - 1 - lo]
                m[dd + NMARG // 2] = lin - pay[k - lo]
        return m


def _put_strip(ctx, f, seg, height):
    """bsm.py:402-440."""
    hi = f + seg.shape[0]
    lo = f - 2 * height - 1
    pay = _payoff(ctx.d["d_s"], lo, hi)
    arr = np.empty(hi - lo + 1, dtype=np.float64)
    arr[: f - lo + 1] = pay[: f - lo + 1]
    arr[f - lo + 1:] = seg
    arr0 = arr.copy() if ctx.want_marg else None
    kb = ctx.sweep(arr, pay, lo, height)
    if arr0 is not None:
        ctx.marg_last = ctx.margins(arr0, pay, lo, height, kb)
    if kb == NONE_SEEN or not f - height <= kb <= f:
        raise OracleError("GeometryError", None)
    return kb, arr[kb + 1 - lo: hi - height - lo + 1].copy()


def _put_solve(ctx, f, seg, h):
    """bsm.py:443-501: boundary recursion on 2h continuation values."""
    if seg.shape[0] != 2 * h:
        raise OracleError("GeometryError", None)
    if h <= ctx.cutoff:
        return _put_strip(ctx, f, seg, h)
    h1 = (h + 1) // 2
    h2 = h - h1
    mid = valid_corr(seg, ctx.power(h1))
    km, upper = _put_solve(ctx, f, seg[: 2 * h1], h1)
    if not f - h1 <= km <= f:
        raise OracleError("GeometryError", None)
    asm = np.concatenate([upper, mid])
    if asm.shape[0] != (f + 2 * h - h1) - km:
        raise OracleError("GeometryError", None)
    bottom = valid_corr(asm, ctx.power(h2))
    kp, lower = _put_solve(ctx, km, asm[: 2 * h2], h2)
    out = np.concatenate([lower, bottom])
    if out.shape[0] != (f + h) - kp:
        raise OracleError("GeometryError", None)
    return kp, out


def put_stage(ctx, f, seg, h):
    """bsm.py:557-582: far jump + near boundary recursion."""
    far = valid_corr(seg, ctx.power(h)) if seg.shape[0] > 2 * h else None
    kp, near = _put_solve(ctx, f, seg[: 2 * h], h)
    out = near if far is None else np.concatenate([near, far])
    if out.shape[0] != (f + seg.shape[0] - h) - kp:
        raise OracleError("GeometryError", None)
    return kp, out


def _put_apex(ctx, f, seg, rem, k_star) -> float:
    """bsm.py:679-713."""
    hi = k_star + rem
    lo = min(f, k_star - rem) - 1
    pay = _payoff(ctx.d["d_s"], lo, hi)
    arr = np.empty(hi - lo + 1, dtype=np.float64)
    if f >= lo:
        arr[: f - lo + 1] = pay[: f - lo + 1]
        arr[f - lo + 1:] = seg
    else:
        arr[:] = seg[lo - (f + 1):]
    ctx.sweep(arr, pay, lo, rem)
    return float(arr[k_star - lo])


def put_fast(S, K, R, Y, V, E, T, lam=0.4, base_cutoff=128, margins=False):
    """bsm.py:585-676: (price, times, cols), plus the per-record boundary
    margins (``boundary_margins``) when ``margins``."""
    if margins:
        return _with_margins(_put_fast, S, K, R, Y, V, E, T, lam, base_cutoff)
    return _put_fast(S, K, R, Y, V, E, T, lam, base_cutoff)[:3]


def _put_fast(S, K, R, Y, V, E, T, lam=0.4, base_cutoff=128, want_marg=False):
    d = discretize_put(S, K, R, Y, V, E, T, lam)
    n, ks = d["n"], d["k_star"]
    if base_cutoff < 1:
        raise OracleError("ValidationError", "base_cutoff")
    if ks <= -n:
        return K - S, np.zeros(1, dtype=np.int64), np.array([min(0, ks + n)], dtype=np.int64)
    if n <= 2 * base_cutoff:
        return put_baseline(S, K, R, Y, V, E, T, lam)
    ctx = _PutCtx(d, base_cutoff)
    ctx.want_marg = want_marg
    times, cols, marg = [0], [0], [_NOMARG]
    m, f = 0, 0
    if ks + n < 1:
        raise OracleError("DomainError", "width")
    seg = np.zeros(ks + n, dtype=np.float64)
    while True:
        rem = n - m
        red = seg.shape[0]
        if red != (ks + rem) - f:
            raise OracleError("GeometryError", None)
        if red == 0:
            price = K * (1.0 - math.exp(ks * d["d_s"]))
            break
        if rem <= 2 * base_cutoff:
            price = K * _put_apex(ctx, f, seg, rem, ks)
            break
        h = min(rem // 2, red // 2)
        ctx.marg_last = None
        if h < 1:
            f, seg = _put_strip(ctx, f, seg, 1)
            m += 1
        else:
            f, seg = put_stage(ctx, f, seg, h)
            m += h
        times.append(m)
        cols.append(f)
        marg.append(_NOMARG if ctx.marg_last is None else ctx.marg_last)
    t = np.asarray(times, dtype=np.int64)
    c = np.asarray(cols, dtype=np.int64)
    order = np.argsort(t)
    return price, t[order], c[order], np.asarray(marg)[order]


def _with_margins(fn, *args):
    """Run a fast pricer with margin recording; early-dispatch results (and
    baseline delegation) carry NaN margins -- no tie slack."""
    out = fn(*args, want_marg=True)
    if len(out) == 4:
        return out
    p, t, c = out
    return p, t, c, np.full((len(t), NMARG), np.nan)


# ---------------------------------------------------------------------------
# dispatch helper used by tests / bench


def price(kind: str, S, K, R, Y, V, E, T, lam=0.4, call_cutoff=256, put_cutoff=128):
    """Fast-path price of one option: kind in {'euro', 'call', 'put'}."""
    if kind == "euro":
        return euro_fast(S, K, R, Y, V, E, T)
    if kind == "call":
        return call_fast(S, K, R, Y, V, E, T, call_cutoff)[0]
    if kind == "put":
        return put_fast(S, K, R, Y, V, E, T, lam, put_cutoff)[0]
    raise ValueError(kind)
