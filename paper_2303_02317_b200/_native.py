"""ctypes binding of ``libfftlattice_b200.so`` (the C ABI in include/fftlattice_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
usable, every pricing call raises.  Batched entry points take and return numpy
arrays (host memory); device buffers are owned by the library.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .model import (
    DomainError,
    GeometryError,
    NumericalIntegrityError,
    PricingError,
    StabilityError,
    ValidationError,
)

__all__ = [
    "KIND_EURO", "KIND_CALL", "KIND_PUT", "METHOD_FAST", "METHOD_BASELINE",
    "lib", "lib_path", "BatchResult", "price_batch", "DeviceBatch", "apply_linear_steps",
    "status_error", "EXPORTED_SYMBOLS", "NativeLibraryError",
]

KIND_EURO, KIND_CALL, KIND_PUT = 0, 1, 2
METHOD_FAST, METHOD_BASELINE, METHOD_GAUSS, METHOD_CLOSED = 0, 1, 2, 3

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_NAME = "libfftlattice_b200.so"
_lock = threading.Lock()
_lib = None

#: Every symbol include/fftlattice_b200.h declares.
EXPORTED_SYMBOLS = (
    "fl_version", "fl_last_error", "fl_price_batch", "fl_batch_prepare", "fl_batch_run", "fl_batch_device_bytes",
    "fl_batch_fetch", "fl_batch_launches", "fl_batch_stats", "fl_batch_profile", "fl_batch_timeline", "fl_batch_free",
    "fl_batch_ref_flops", "fl_inspect", "fl_apply_linear_steps", "fl_put_trapezoid", "fl_call_trapezoid",
    "fl_call_grid", "fl_put_march_rows", "fl_put_fast_rows", "fl_fft", "fl_convolve", "fl_euro_approx",
    "fl_probe_fp64", "fl_release_cache", "fl_shard_plan", "fl_price_batch_multi", "fl_price_batch_dev",
    "fl_price_put_bsm", "fl_price_american_call", "fl_price_european", "fl_dev_workspace_bytes", "fl_sync",
    "fl_release_dev_cache", "fl_kernel_power", "fl_price_batch_ex", "fl_probe_transcendentals",
)


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing or a library call failed (not a pricing error)."""


def lib_path() -> str:
    return os.path.join(HERE, _LIB_NAME)


def lib():
    """Load the CUDA library (raises NativeLibraryError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{path} is not built; run `python -m paper_2303_02317_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(path)
        P, i64, i32, d, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_int
        L.fl_version.restype = c_int
        L.fl_last_error.restype = ctypes.c_char_p
        L.fl_price_batch.argtypes = [i64, P, P, P, P, P, P, P, P, d, i64, i64, c_int, P, P, P, P, P, i32, P]
        L.fl_price_batch.restype = c_int
        L.fl_batch_prepare.argtypes = [ctypes.POINTER(P), i64, P, P, P, P, P, P, P, P, d, i64, i64, c_int, i32, P]
        L.fl_batch_prepare.restype = c_int
        L.fl_batch_run.argtypes = [P, P]
        L.fl_batch_run.restype = c_int
        L.fl_batch_fetch.argtypes = [P, P, P, P, P, P, P]
        L.fl_batch_fetch.restype = c_int
        L.fl_batch_launches.argtypes = [P]
        L.fl_batch_launches.restype = c_int
        L.fl_batch_device_bytes.argtypes = [P]
        L.fl_batch_device_bytes.restype = ctypes.c_int64
        L.fl_batch_free.argtypes = [P]
        L.fl_batch_free.restype = None
        L.fl_apply_linear_steps.argtypes = [P, i64, c_int, d, d, d, i64, P, P]
        L.fl_apply_linear_steps.restype = c_int
        L.fl_batch_stats.argtypes = [P, P, P, P, P]
        L.fl_batch_stats.restype = c_int
        L.fl_batch_profile.argtypes = [P, P, P]
        L.fl_batch_profile.restype = c_int
        L.fl_batch_timeline.argtypes = [P, P, P]
        L.fl_batch_timeline.restype = c_int
        L.fl_inspect.argtypes = [i64, P, P, P, P, P, P, P, P, d, i64, i64, P, P, P, P]
        L.fl_inspect.restype = c_int
        L.fl_batch_ref_flops.argtypes = [P, P, P]
        L.fl_batch_ref_flops.restype = c_int
        L.fl_put_trapezoid.argtypes = [d, d, d, d, i64, i64, P, i64, i64, P, P, P, P]
        L.fl_put_trapezoid.restype = c_int
        L.fl_call_trapezoid.argtypes = [d, d, d, d, d, i64, i64, i64, i64, P, i64, P, P, P, P]
        L.fl_call_trapezoid.restype = c_int
        L.fl_call_grid.argtypes = [d, d, d, d, d, i64, P, P, P, P, P]
        L.fl_call_grid.restype = c_int
        L.fl_put_march_rows.argtypes = [d, d, d, d, d, i64, i64, P, c_int, P, i64, P, P, P]
        L.fl_put_march_rows.restype = c_int
        L.fl_put_fast_rows.argtypes = [d, d, d, d, d, i64, d, i64, P, i64, P, P, P, P, P, P, i32, P]
        L.fl_put_fast_rows.restype = c_int
        L.fl_fft.argtypes = [P, i64, c_int, P, P]
        L.fl_fft.restype = c_int
        L.fl_convolve.argtypes = [P, i64, P, i64, P, P]
        L.fl_convolve.restype = c_int
        L.fl_euro_approx.argtypes = [i64, P, P, P, P, P, P, P, c_int, P, P, P]
        L.fl_euro_approx.restype = c_int
        L.fl_probe_fp64.argtypes = [P, P]
        L.fl_probe_fp64.restype = c_int
        L.fl_probe_transcendentals.argtypes = [P, P, P]
        L.fl_probe_transcendentals.restype = c_int
        L.fl_release_cache.argtypes = []
        L.fl_release_cache.restype = None
        L.fl_release_dev_cache.argtypes = []
        L.fl_release_dev_cache.restype = None
        L.fl_shard_plan.argtypes = [i64, P, P, c_int, P]
        L.fl_shard_plan.restype = c_int
        L.fl_price_batch_multi.argtypes = [c_int, P, i64, P, P, P, P, P, P, P, P, d, i64, i64, c_int,
                                           P, P, P, P, P, i32]
        L.fl_price_batch_multi.restype = c_int
        L.fl_price_batch_dev.argtypes = [i64, P, c_int, P, P, P, P, P, P, P, d, i64, i64, c_int, i64,
                                         P, P, P, P, P, i32, P]
        L.fl_price_batch_dev.restype = c_int
        L.fl_price_put_bsm.argtypes = [i64, P, P, P, P, P, P, P, d, i64, i64, P, P, P, P, P, i32, P]
        L.fl_price_put_bsm.restype = c_int
        L.fl_price_american_call.argtypes = [i64, P, P, P, P, P, P, P, i64, i64, P, P, P, P, P, i32, P]
        L.fl_price_american_call.restype = c_int
        L.fl_price_european.argtypes = [i64, P, P, P, P, P, P, P, P, P, P]
        L.fl_price_european.restype = c_int
        L.fl_dev_workspace_bytes.argtypes = [i64, i64, c_int, i64, i64, P]
        L.fl_dev_workspace_bytes.restype = c_int
        L.fl_sync.argtypes = [P]
        L.fl_sync.restype = c_int
        L.fl_price_batch_ex.argtypes = [i64, P, P, P, P, P, P, P, P, P, d, i64, i64, c_int, P, P, P, P, P, i32, P]
        L.fl_price_batch_ex.restype = c_int
        L.fl_kernel_power.argtypes = [P, i64, i64, P, P]
        L.fl_kernel_power.restype = c_int
        _lib = L
        return L


def _check(rc: int) -> None:
    if rc != 0:
        raise NativeLibraryError(lib().fl_last_error().decode(errors="replace"))


def _f64(a, n):
    out = np.ascontiguousarray(np.broadcast_to(np.asarray(a, dtype=np.float64), (n,)))
    return out


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# status codes (csrc/fl_status.h)

_FIELDS = {1: "spot", 2: "strike", 3: "rate", 4: "dividend_yield", 5: "volatility",
           6: "days_to_expiry", 7: "steps", 8: "prob_up", 9: "lam", 10: "base_cutoff", 11: "times"}
_FIELD_MSG = {
    "spot": "spot must be positive and finite",
    "strike": "strike must be nonnegative and finite",
    "rate": "rate must be nonnegative and finite",
    "dividend_yield": "dividend_yield must be nonnegative and finite",
    "volatility": "volatility must be positive",
    "days_to_expiry": "days_to_expiry must be positive",
    "steps": "steps must be >= 1",
    "prob_up": "prob_up out of (0, 1): the carry outruns one lattice step; "
               "increase steps or volatility",
    "lam": "lambda must be positive",
    "base_cutoff": "base_cutoff must be >= 1",
    "times": "times must be strictly increasing",
}
_WEIGHTS = {1: ("coef_mid", "centre weight is negative; choose a smaller lambda"),
            2: ("coef_up", "upper weight is negative; increase steps or adjust lambda"),
            3: ("coef_down", "lower weight is negative; increase steps or adjust lambda")}


def status_error(code: int) -> Exception | None:
    """Exception instance equivalent to the reference's for a status code."""
    code = int(code)
    if code == 0:
        return None
    cls, det = code & 0xFF00, code & 0xFF
    if cls == 0x100:
        f = _FIELDS.get(det, "unknown")
        return ValidationError(f, _FIELD_MSG.get(f, f))
    if cls == 0x200:
        w, msg = _WEIGHTS.get(det, ("unknown", "negative weight"))
        return StabilityError(w, msg)
    if cls == 0x300:
        if det == 1:
            return DomainError("spot lies too many grid nodes from the strike")
        if det == 3:
            return DomainError("degenerate Gaussian weight window")
        if det == 4:
            return DomainError("strike must be positive for the closed form")
        return DomainError("put grid requires a positive strike")
    if cls == 0x400:
        return GeometryError(f"decomposition failed to tile its region (site {det})")
    if cls == 0x500:
        return NumericalIntegrityError("numerical self-check failed")
    if cls == 0x600:
        return ValueError("math domain error")
    return PricingError(f"unsupported on this GPU build (status {code:#x})")


# --------------------------------------------------------------------------
# batched pricing


class BatchResult:
    """Per-option outputs of a batched call (numpy, host)."""

    def __init__(self, price, status, bt, bc, bcount, cap):
        self.price, self.status = price, status
        self.bnd_times, self.bnd_cols, self.bnd_count, self.cap = bt, bc, bcount, cap

    def boundary(self, i: int):
        c = int(self.bnd_count[i])
        if c > self.cap:
            raise IndexError("boundary record truncated; re-run with a larger bnd_cap")
        return self.bnd_times[i, :c].copy(), self.bnd_cols[i, :c].copy()


def _inputs(kind, S, K, R, Y, V, E, T):
    n = int(np.asarray(S).shape[0]) if np.ndim(S) else 1
    k = np.ascontiguousarray(np.broadcast_to(np.asarray(kind, dtype=np.int8), (n,)))
    t = np.ascontiguousarray(np.broadcast_to(np.asarray(T, dtype=np.int64), (n,)))
    return n, k, _f64(S, n), _f64(K, n), _f64(R, n), _f64(Y, n), _f64(V, n), _f64(E, n), t


def price_batch(kind, S, K, R, Y, V, E, T, *, lam=0.4, call_cutoff=256, put_cutoff=128,
                method=METHOD_FAST, bnd_cap=0, stream=None, bparams=None) -> BatchResult:
    """Price a batch through ``fl_price_batch`` (host arrays in and out);
    ``bparams`` (n x 4: weight_down, weight_up, log_up, step_years; NaN rows
    derive) overrides the binomial lattice constants (``fl_price_batch_ex``)."""
    n, k, S, K, R, Y, V, E, T = _inputs(kind, S, K, R, Y, V, E, T)
    price = np.empty(n)
    status = np.empty(n, dtype=np.int32)
    cap = int(bnd_cap)
    bt = np.empty((n, max(cap, 1)), dtype=np.int64)
    bc = np.empty((n, max(cap, 1)), dtype=np.int64)
    bcount = np.zeros(n, dtype=np.int32)
    bp = None if bparams is None else np.ascontiguousarray(np.broadcast_to(
        np.asarray(bparams, dtype=np.float64), (n, 4)))
    _check(lib().fl_price_batch_ex(
        n, _ptr(k), _ptr(S), _ptr(K), _ptr(R), _ptr(Y), _ptr(V), _ptr(E), _ptr(T),
        _ptr(bp) if bp is not None else None, float(lam),
        int(call_cutoff), int(put_cutoff), int(method), _ptr(price), _ptr(status),
        _ptr(bt) if cap else None, _ptr(bc) if cap else None, _ptr(bcount) if cap else None,
        cap, ctypes.c_void_p(stream) if stream else None))
    return BatchResult(price, status, bt, bc, bcount, cap)


class DeviceBatch:
    """A prepared, device-resident batch (``fl_batch_prepare`` / run / fetch)."""

    def __init__(self, kind, S, K, R, Y, V, E, T, *, lam=0.4, call_cutoff=256, put_cutoff=128,
                 method=METHOD_FAST, bnd_cap=0, stream=None):
        n, k, S, K, R, Y, V, E, T = _inputs(kind, S, K, R, Y, V, E, T)
        self.n, self.cap = n, int(bnd_cap)
        h = ctypes.c_void_p()
        _check(lib().fl_batch_prepare(
            ctypes.byref(h), n, _ptr(k), _ptr(S), _ptr(K), _ptr(R), _ptr(Y), _ptr(V), _ptr(E), _ptr(T),
            float(lam), int(call_cutoff), int(put_cutoff), int(method), self.cap,
            ctypes.c_void_p(stream) if stream else None))
        self._h = h

    def run(self, stream=None) -> None:
        _check(lib().fl_batch_run(self._h, ctypes.c_void_p(stream) if stream else None))

    def profile(self, stream=None) -> np.ndarray:
        """Scheduler profile counters of the last run (FL_PROFILE=1 at run time)."""
        out = np.zeros(56, dtype=np.uint64)
        _check(lib().fl_batch_profile(self._h, _ptr(out), ctypes.c_void_p(stream) if stream else None))
        return out

    def timeline(self, stream=None) -> np.ndarray:
        """(n, 3) per work item of the last run: start ns, end ns, SM << 1 | chain (FL_PROFILE=1)."""
        out = np.zeros((self.n, 3), dtype=np.uint64)
        _check(lib().fl_batch_timeline(self._h, _ptr(out), ctypes.c_void_p(stream) if stream else None))
        return out

    def launches(self) -> int:
        return int(lib().fl_batch_launches(self._h))

    def device_bytes(self) -> int:
        """Device memory this batch holds (fl_batch_device_bytes)."""
        v = int(lib().fl_batch_device_bytes(self._h))
        if v < 0:
            raise NativeLibraryError(lib().fl_last_error().decode())
        return v

    def stats(self, stream=None) -> dict:
        """Executed fp64 flops of the last run and the H2D / D2H bytes moved."""
        f = ctypes.c_double(0.0)
        hb, db = ctypes.c_int64(0), ctypes.c_int64(0)
        _check(lib().fl_batch_stats(self._h, ctypes.byref(f), ctypes.byref(hb), ctypes.byref(db),
                                    ctypes.c_void_p(stream) if stream else None))
        r = ctypes.c_double(0.0)
        _check(lib().fl_batch_ref_flops(self._h, ctypes.byref(r), ctypes.c_void_p(stream) if stream else None))
        return {"fp64_flops": f.value, "ref_flops": r.value, "h2d_bytes": hb.value, "d2h_bytes": db.value}

    def fetch(self, stream=None) -> BatchResult:
        n, cap = self.n, self.cap
        price = np.empty(n)
        status = np.empty(n, dtype=np.int32)
        bt = np.empty((n, max(cap, 1)), dtype=np.int64)
        bc = np.empty((n, max(cap, 1)), dtype=np.int64)
        bcount = np.zeros(n, dtype=np.int32)
        _check(lib().fl_batch_fetch(self._h, _ptr(price), _ptr(status), _ptr(bt) if cap else None,
                                    _ptr(bc) if cap else None, _ptr(bcount) if cap else None,
                                    ctypes.c_void_p(stream) if stream else None))
        return BatchResult(price, status, bt, bc, bcount, cap)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().fl_batch_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def apply_linear_steps(x: np.ndarray, taps: int, c0: float, c1: float, c2: float, h: int) -> np.ndarray:
    """Valid-mode correlation of x with the h-th composed stencil, on device."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(x.shape[0] - h * (taps - 1))
    _check(lib().fl_apply_linear_steps(_ptr(x), x.shape[0], int(taps), float(c0), float(c1),
                                       float(c2), int(h), _ptr(out), None))
    return out


def price_batch_full(kind, S, K, R, Y, V, E, T, *, lam=0.4, call_cutoff=256, put_cutoff=128,
                     method=METHOD_FAST, bnd_cap=64, stream=None, bparams=None) -> BatchResult:
    """``price_batch`` with complete boundary records: options whose record
    exceeded ``bnd_cap`` are re-run with a capacity that fits them."""
    res = price_batch(kind, S, K, R, Y, V, E, T, lam=lam, call_cutoff=call_cutoff, put_cutoff=put_cutoff,
                      method=method, bnd_cap=bnd_cap, stream=stream, bparams=bparams)
    over = np.nonzero(res.bnd_count > res.cap)[0]
    if over.size == 0:
        return res
    n, k, S, K, R, Y, V, E, T = _inputs(kind, S, K, R, Y, V, E, T)
    cap2 = int(res.bnd_count[over].max())
    sub = price_batch(k[over], S[over], K[over], R[over], Y[over], V[over], E[over], T[over], lam=lam,
                      call_cutoff=call_cutoff, put_cutoff=put_cutoff, method=method, bnd_cap=cap2,
                      stream=stream,
                      bparams=None if bparams is None else np.broadcast_to(np.asarray(bparams), (n, 4))[over])
    bt = np.full((n, cap2), 0, dtype=np.int64)
    bc = np.full((n, cap2), 0, dtype=np.int64)
    c0 = res.cap
    bt[:, :c0] = res.bnd_times[:, :c0]
    bc[:, :c0] = res.bnd_cols[:, :c0]
    bt[over] = sub.bnd_times
    bc[over] = sub.bnd_cols
    price, status, bcount = res.price.copy(), res.status.copy(), res.bnd_count.copy()
    price[over], status[over], bcount[over] = sub.price, sub.status, sub.bnd_count
    return BatchResult(price, status, bt, bc, bcount, cap2)


def probe_fp64_tflops(stream=None) -> float:
    """Measured DFMA throughput of the current device (TFLOP/s)."""
    t = ctypes.c_double(0.0)
    _check(lib().fl_probe_fp64(ctypes.byref(t), ctypes.c_void_p(stream) if stream else None))
    return t.value


def probe_transcendentals(stream=None):
    """(exp, log) fp64 evaluations per second on the current device."""
    a, b = ctypes.c_double(0.0), ctypes.c_double(0.0)
    _check(lib().fl_probe_transcendentals(ctypes.byref(a), ctypes.byref(b), ctypes.c_void_p(stream) if stream else None))
    return a.value, b.value


def put_trapezoid(cd: float, cm: float, cu: float, ds: float, base_cutoff: int, f: int, seg: np.ndarray, h: int):
    """fl_put_trapezoid: (new boundary, values of cols kp+1 .. f+W-h); raises on a status."""
    seg = np.ascontiguousarray(seg, dtype=np.float64)
    W = int(seg.shape[0])
    out = np.empty(W + h)
    kp = ctypes.c_int64(0)
    st = ctypes.c_int32(0)
    _check(lib().fl_put_trapezoid(float(cd), float(cm), float(cu), float(ds), int(base_cutoff), int(f), _ptr(seg),
                                  W, int(h), _ptr(out), ctypes.byref(kp), ctypes.byref(st), None))
    err = status_error(st.value)
    if err is not None:
        raise err
    n_out = (f + W - h) - kp.value
    return kp.value, out[:n_out].copy()


def call_trapezoid(S: float, K: float, wd: float, wu: float, lu: float, base_cutoff: int, i: int, j: int,
                   first: int, run: np.ndarray, h: int):
    """fl_call_trapezoid: (new boundary jp, red values of cols first .. jp); raises on a status."""
    run = np.ascontiguousarray(run, dtype=np.float64)
    out = np.empty(max(int(run.shape[0]), 1))
    jp = ctypes.c_int64(0)
    st = ctypes.c_int32(0)
    _check(lib().fl_call_trapezoid(float(S), float(K), float(wd), float(wu), float(lu), int(base_cutoff), int(i),
                                   int(j), int(first), _ptr(run), int(h), _ptr(out), ctypes.byref(jp),
                                   ctypes.byref(st), None))
    err = status_error(st.value)
    if err is not None:
        raise err
    return jp.value, out[:max(jp.value - first + 1, 0)].copy()


def inspect(kind, S, K, R, Y, V, E, T, *, lam=0.4, call_cutoff=256, put_cutoff=128):
    """Host-only derivation the batch entry points perform (fl_inspect):
    (status[n], mode[n], dparams[n, 4], iparams[n, 2]).  No CUDA involved."""
    n, k, S, K, R, Y, V, E, T = _inputs(kind, S, K, R, Y, V, E, T)
    status = np.zeros(n, dtype=np.int32)
    mode = np.zeros(n, dtype=np.int32)
    dp = np.zeros((n, 4))
    ip = np.zeros((n, 2), dtype=np.int64)
    _check(lib().fl_inspect(n, _ptr(k), _ptr(S), _ptr(K), _ptr(R), _ptr(Y), _ptr(V), _ptr(E), _ptr(T), float(lam),
                            int(call_cutoff), int(put_cutoff), _ptr(status), _ptr(mode), _ptr(dp), _ptr(ip)))
    return status, mode, dp, ip


def call_grid(S, K, wd, wu, lu, n):
    """fl_call_grid: (price, rows list, masks list, first-green cols)."""
    n = int(n)
    cells = (n + 1) * (n + 2) // 2
    rows = np.empty(cells)
    masks = np.empty(cells, dtype=np.uint8)
    cols = np.empty(n + 1, dtype=np.int64)
    price = ctypes.c_double(0.0)
    _check(lib().fl_call_grid(float(S), float(K), float(wd), float(wu), float(lu), n, _ptr(rows), _ptr(masks),
                              _ptr(cols), ctypes.byref(price), None))
    rl = [rows[i * (i + 1) // 2: i * (i + 1) // 2 + i + 1].copy() for i in range(n + 1)]
    ml = [masks[i * (i + 1) // 2: i * (i + 1) // 2 + i + 1].astype(bool) for i in range(n + 1)]
    return price.value, rl, ml, cols


def put_march_rows(cd, cm, cu, ds, K, ks, n, times):
    """fl_put_march_rows: (price, last_green cols[0..n], {t: window values})."""
    n = int(n)
    times = np.ascontiguousarray(sorted(set(int(t) for t in times)), dtype=np.int64)
    cap = int(sum(2 * n + 1 - 2 * t for t in times))
    snap = np.empty(max(cap, 1))
    lg = np.empty(n + 1, dtype=np.int64)
    price = ctypes.c_double(0.0)
    _check(lib().fl_put_march_rows(float(cd), float(cm), float(cu), float(ds), float(K), int(ks), n,
                                   _ptr(times) if len(times) else None, len(times), _ptr(snap), cap, _ptr(lg),
                                   ctypes.byref(price), None))
    out, off = {}, 0
    for t in times.tolist():
        m = 2 * n + 1 - 2 * t
        out[t] = snap[off:off + m].copy()
        off += m
    return price.value, lg, out


def put_fast_rows(S, K, R, V, E, T, lam, base_cutoff):
    """fl_put_fast_rows: (price, status, times, cols, flat snapshot buffer)."""
    cap = 1 << 16
    for _ in range(3):
        snap = np.empty(cap)
        used = ctypes.c_int64(0)
        price = ctypes.c_double(0.0)
        status = ctypes.c_int32(0)
        bcap = 128
        bt = np.empty(bcap, dtype=np.int64)
        bc = np.empty(bcap, dtype=np.int64)
        bn = ctypes.c_int32(0)
        _check(lib().fl_put_fast_rows(float(S), float(K), float(R), float(V), float(E), int(T), float(lam),
                                      int(base_cutoff), _ptr(snap), cap, ctypes.byref(used), ctypes.byref(price),
                                      ctypes.byref(status), _ptr(bt), _ptr(bc), ctypes.byref(bn), bcap, None))
        if used.value <= cap:
            k = min(bn.value, bcap)
            return price.value, status.value, bt[:k].copy(), bc[:k].copy(), snap[:used.value].copy()
        cap = int(used.value) + 16
    raise NativeLibraryError("fl_put_fast_rows: snapshot buffer did not converge")


def fft(vec: np.ndarray, inverse: bool) -> np.ndarray:
    """fl_fft on a complex128 vector (power-of-two length)."""
    v = np.ascontiguousarray(vec, dtype=np.complex128)
    out = np.empty_like(v)
    _check(lib().fl_fft(_ptr(v), v.shape[0], 1 if inverse else 0, _ptr(out), None))
    return out


def convolve(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """fl_convolve on complex128 vectors: full linear convolution."""
    a = np.ascontiguousarray(x, dtype=np.complex128)
    b = np.ascontiguousarray(y, dtype=np.complex128)
    out = np.empty(a.shape[0] + b.shape[0] - 1, dtype=np.complex128)
    _check(lib().fl_convolve(_ptr(a), a.shape[0], _ptr(b), b.shape[0], _ptr(out), None))
    return out


def euro_approx(S, K, R, Y, V, E, T, method):
    """fl_euro_approx: (price, status) for METHOD_GAUSS / METHOD_CLOSED."""
    n, _, S, K, R, Y, V, E, T = _inputs(0, S, K, R, Y, V, E, T)
    price = np.empty(n)
    status = np.empty(n, dtype=np.int32)
    _check(lib().fl_euro_approx(n, _ptr(S), _ptr(K), _ptr(R), _ptr(Y), _ptr(V), _ptr(E), _ptr(T), int(method),
                                _ptr(price), _ptr(status), None))
    return price, status


# --------------------------------------------------------------------------
# multi-device and device-pointer entry points


def shard_plan(kind, T, nshard: int) -> np.ndarray:
    """fl_shard_plan: owner shard of every option (LPT over the cost model)."""
    k = np.ascontiguousarray(np.asarray(kind, dtype=np.int8))
    t = np.ascontiguousarray(np.broadcast_to(np.asarray(T, dtype=np.int64), k.shape))
    owner = np.empty(k.shape[0], dtype=np.int32)
    _check(lib().fl_shard_plan(k.shape[0], _ptr(k), _ptr(t), int(nshard), _ptr(owner)))
    return owner


def price_batch_multi(kind, S, K, R, Y, V, E, T, *, devices=None, lam=0.4, call_cutoff=256, put_cutoff=128,
                      method=METHOD_FAST, bnd_cap=0) -> BatchResult:
    """One call over several GPUs (fl_price_batch_multi): LPT shards, one host
    thread and stream per device, results gathered into host arrays."""
    if devices is None:
        import torch

        devices = list(range(torch.cuda.device_count()))
    devs = np.ascontiguousarray(np.asarray(devices, dtype=np.int32))
    n, k, S, K, R, Y, V, E, T = _inputs(kind, S, K, R, Y, V, E, T)
    price = np.empty(n)
    status = np.empty(n, dtype=np.int32)
    cap = int(bnd_cap)
    bt = np.empty((n, max(cap, 1)), dtype=np.int64)
    bc = np.empty((n, max(cap, 1)), dtype=np.int64)
    bcount = np.zeros(n, dtype=np.int32)
    _check(lib().fl_price_batch_multi(
        int(devs.shape[0]), _ptr(devs), n, _ptr(k), _ptr(S), _ptr(K), _ptr(R), _ptr(Y), _ptr(V), _ptr(E),
        _ptr(T), float(lam), int(call_cutoff), int(put_cutoff), int(method), _ptr(price), _ptr(status),
        _ptr(bt) if cap else None, _ptr(bc) if cap else None, _ptr(bcount) if cap else None, cap))
    return BatchResult(price, status, bt, bc, bcount, cap)


def _dptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def price_batch_dev(kind, S, K, R, Y, V, E, T, *, max_steps=None, lam=0.4, call_cutoff=256, put_cutoff=128,
                    method=METHOD_FAST, bnd_cap=0, kind_all=None, stream=None):
    """fl_price_batch_dev on torch CUDA tensors (caller-owned device buffers).

    Inputs: float64 S..E, int64 T, int8 ``kind`` (or ``kind=None`` with
    ``kind_all``), all on one CUDA device.  Returns torch tensors
    ``(price, status)`` (plus ``(bnd_times, bnd_cols, bnd_count)`` when
    ``bnd_cap > 0``), enqueued on ``stream`` (default: torch's current stream)
    with no synchronization.  ``max_steps`` sizes the workspaces; when omitted
    it is read from ``T`` (one device-to-host read)."""
    import torch

    dev = S.device
    n = int(S.shape[0])
    cols = []
    for x, dt in ((S, torch.float64), (K, torch.float64), (R, torch.float64), (Y, torch.float64),
                  (V, torch.float64), (E, torch.float64), (T, torch.int64)):
        if x.device != dev or x.dtype != dt or not x.is_contiguous():
            raise ValueError("price_batch_dev: inputs must be contiguous tensors of one CUDA device "
                             "(float64 S..E, int64 T)")
        cols.append(x)
    if kind is not None and (kind.dtype != torch.int8 or kind.device != dev):
        raise ValueError("price_batch_dev: kind must be an int8 tensor on the inputs' device")
    if kind is None and kind_all is None:
        raise ValueError("price_batch_dev: pass kind or kind_all")
    if max_steps is None:
        max_steps = int(T.max().item()) if n else 1
    price = torch.empty(n, dtype=torch.float64, device=dev)
    status = torch.empty(n, dtype=torch.int32, device=dev)
    cap = int(bnd_cap)
    bt = torch.empty((n, cap), dtype=torch.int64, device=dev) if cap else None
    bc = torch.empty((n, cap), dtype=torch.int64, device=dev) if cap else None
    bn = torch.zeros(n, dtype=torch.int32, device=dev) if cap else None
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        _check(lib().fl_price_batch_dev(
            n, _dptr(kind), -1 if kind_all is None else int(kind_all), *(_dptr(c) for c in cols), float(lam),
            int(call_cutoff), int(put_cutoff), int(method), int(max_steps), _dptr(price), _dptr(status),
            _dptr(bt), _dptr(bc), _dptr(bn), cap, ctypes.c_void_p(stream) if stream else None))
    if cap:
        return price, status, bt, bc, bn
    return price, status


def dev_workspace_bytes(n: int, max_steps: int, method=METHOD_FAST, call_cutoff=256, put_cutoff=128) -> int:
    b = ctypes.c_int64(0)
    _check(lib().fl_dev_workspace_bytes(int(n), int(max_steps), int(method), int(call_cutoff), int(put_cutoff),
                                        ctypes.byref(b)))
    return b.value


def release_caches() -> None:
    """Free this thread's cached host-path batches and device-path workspaces."""
    lib().fl_release_cache()
    lib().fl_release_dev_cache()


def kernel_power(weights: np.ndarray, h: int) -> np.ndarray:
    """fl_kernel_power: generic composed kernel (spectrum power on the device)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.empty(int(h) * (w.shape[0] - 1) + 1)
    _check(lib().fl_kernel_power(_ptr(w), w.shape[0], int(h), _ptr(out), None))
    return out
