"""Composed-stencil operators -- drop-in for the hot-path part of ``fftlattice.fft``.

``Kernel`` (fft.py:41-74), ``kernel_power`` (fft.py:203-260) and
``apply_linear_steps`` (fft.py:263-329) with the reference signatures; the
composition and the valid-mode correlation run on the device
(``fl_apply_linear_steps``: truncated overlap-save FFT with the analytic
stencil spectrum, csrc/fl_conv.cuh, for the pricers' own two- / three-tap
nonnegative stencils; ``fl_kernel_power`` + ``fl_convolve``, the device
transform pair, for any other kernel).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .model import (
    GridRow,
    InsufficientWidthError,
    NumericalIntegrityError,
    ValidationError,
)

__all__ = ["Kernel", "kernel_power", "apply_linear_steps", "fft_forward", "fft_inverse", "convolve"]


@dataclass(frozen=True, slots=True)
class Kernel:
    """One-step stencil: out[j] = sum_r weights[r] in[j + min_offset + r] (fft.py:41-74)."""

    weights: np.ndarray
    min_offset: int

    def __post_init__(self) -> None:
        arr = np.ascontiguousarray(self.weights, dtype=np.float64)
        object.__setattr__(self, "weights", arr)
        if arr.ndim != 1 or arr.shape[0] < 1:
            raise ValidationError("weights", "kernel weights must be a nonempty 1-D array")

    def __len__(self) -> int:
        return int(self.weights.shape[0])

    @property
    def max_offset(self) -> int:
        return self.min_offset + len(self) - 1


def _fast_taps(w: np.ndarray) -> bool:
    """The pricers' own stencils: two or three nonnegative finite taps (analytic
    spectrum / direct composed weights on the device, fl_apply_linear_steps)."""
    return len(w) in (2, 3) and bool(np.all(np.isfinite(w))) and bool(np.all(w >= 0.0))


def _device_taps(w: np.ndarray) -> tuple[int, float, float, float]:
    c2 = float(w[2]) if len(w) == 3 else 0.0
    return len(w), float(w[0]), float(w[1]), c2


def _power_core(w: np.ndarray, h: int) -> np.ndarray:
    """Composed weights of a kernel with nonzero first and last taps."""
    if _fast_taps(w):
        taps, c0, c1, c2 = _device_taps(w)
        m = h * (taps - 1) + 1
        x = np.zeros(2 * m - 1)
        x[m - 1] = 1.0
        y = _native.apply_linear_steps(x, taps, c0, c1, c2, h)  # y[k] = W[m-1-k]
        return np.ascontiguousarray(y[::-1])
    return _native.kernel_power(w, h)  # generic: spectrum ** h on the device


def kernel_power(kernel: Kernel, h: int) -> Kernel:
    """h-fold composition of ``kernel`` (fft.py:203-260) on the device.

    Exact zero taps at either end stay exact zeros (fft.py:176-183 for two
    taps: they only shift the composed kernel); the nonzero core is composed
    on the device -- the pricers' two- / three-tap nonnegative stencils as the
    composed correlation of a unit impulse (analytic spectrum), any other
    kernel (more taps, negative weights) by raising its spectrum to the h-th
    power and inverting, as the reference does (fft.py:244-260)."""
    if h < 0:
        raise ValidationError("h", "step count h must be >= 0")
    if h == 0:
        return Kernel(np.array([1.0]), 0)
    if h == 1:
        return Kernel(kernel.weights.copy(), kernel.min_offset)
    w = kernel.weights
    out_len = h * (len(w) - 1) + 1
    if not np.all(np.isfinite(w)):
        raise NumericalIntegrityError(f"composed kernel overflowed for h={h}")
    nz = np.nonzero(w)[0]
    out = np.zeros(out_len)
    if nz.size:
        lead = int(nz[0])
        core = _power_core(np.ascontiguousarray(w[lead:int(nz[-1]) + 1]), h)
        out[h * lead:h * lead + core.shape[0]] = core
    if not np.all(np.isfinite(out)):
        raise NumericalIntegrityError(
            f"composed kernel overflowed for h={h} (max weight magnitude {np.max(np.abs(w)):.3e})")
    return Kernel(out, h * kernel.min_offset)


def apply_linear_steps(row: GridRow, kernel: Kernel, h: int, *, direction: int = 1,
                       composed: Kernel | None = None) -> GridRow:
    """Advance ``row`` by h linear steps in one device correlation (fft.py:263-329).

    The pricers' stencils (two / three nonnegative taps) run the device
    correlation with the analytic spectrum (direct composed weights for
    h <= 64); any other kernel is composed by ``kernel_power`` (or taken from
    ``composed``, the reference's cache hook) and correlated by the device
    transform pair, the reference's own route (fft.py:302-329)."""
    if h < 0:
        raise ValidationError("h", "step count h must be >= 0")
    if h == 0:
        return GridRow(row.time_index, row.col_offset, row.values.copy())
    expected_len = h * (len(kernel) - 1) + 1
    if composed is not None and len(composed) != expected_len:
        raise ValidationError("composed", "composed kernel length does not match h steps")
    out_len = len(row) - expected_len + 1
    if out_len < 1:
        raise InsufficientWidthError(
            f"run of {len(row)} columns is too narrow for {h} steps of a "
            f"{len(kernel)}-point kernel (needs >= {expected_len})")
    if _fast_taps(kernel.weights):
        taps, c0, c1, c2 = _device_taps(kernel.weights)
        vals = _native.apply_linear_steps(row.values, taps, c0, c1, c2, h)
    else:
        ck = composed if composed is not None else kernel_power(kernel, h)
        full = _native.convolve(row.values.astype(np.float64), np.ascontiguousarray(ck.weights[::-1]))
        vals = np.ascontiguousarray(full.real[expected_len - 1:len(row)])
    return GridRow(row.time_index + direction * h, row.col_offset - h * kernel.min_offset, vals)


def _require_pow2(n: int) -> None:
    if n < 1 or (n & (n - 1)) != 0:
        raise ValidationError("length", f"fft length must be a power of two, got {n}")


def fft_forward(vec: np.ndarray) -> np.ndarray:
    """Unnormalised DFT of a power-of-two vector on the device (fft.py:84-111)."""
    arr = np.asarray(vec)
    if arr.ndim != 1:
        raise ValidationError("vec", "fft input must be 1-D")
    _require_pow2(arr.shape[0])
    return _native.fft(arr, inverse=False)


def fft_inverse(vec: np.ndarray) -> np.ndarray:
    """Inverse DFT with the 1/N factor on the device (fft.py:114-123)."""
    arr = np.asarray(vec)
    if arr.ndim != 1:
        raise ValidationError("vec", "fft input must be 1-D")
    _require_pow2(arr.shape[0])
    return _native.fft(arr, inverse=True)


def convolve(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Full linear convolution by the transform pair on the device (fft.py:130-163).
    Real inputs give a real float64 result, complex inputs the complex one."""
    ax = np.asarray(x)
    ay = np.asarray(y)
    if ax.ndim != 1 or ay.ndim != 1 or ax.shape[0] < 1 or ay.shape[0] < 1:
        raise ValidationError("x", "convolve inputs must be nonempty 1-D")
    out = _native.convolve(ax, ay)
    if not (np.iscomplexobj(x) or np.iscomplexobj(y)):
        return np.ascontiguousarray(out.real)
    return out
