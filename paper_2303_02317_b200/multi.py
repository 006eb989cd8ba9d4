"""Multi-GPU pricing in one call: every option is independent,
so a batch is LPT-sharded over the box's GPUs by the per-option cost model
(``fl_shard_plan``), each shard is priced by its own host thread on its own
device and stream inside the library (``fl_price_batch_multi``, C++
std::thread per device), and the results are scattered back -- no collective
on the data path.  Replaces the reference's sequential portfolio loop
(cli.py:820-841).  Per-option arithmetic never depends on the shard, so the
result is bit-identical to a single-device ``price_batch``.
"""

from __future__ import annotations

import numpy as np

from . import _native

__all__ = ["price_batch_multi"]


def price_batch_multi(kind, S, K, R, Y, V, E, T, *, devices=None, lam=0.4, call_cutoff=256, put_cutoff=128,
                      method=_native.METHOD_FAST):
    """(price, status) numpy arrays for a mixed batch priced over ``devices``
    (default: every visible CUDA device)."""
    res = _native.price_batch_multi(kind, S, K, R, Y, V, E, T, devices=devices, lam=lam,
                                    call_cutoff=call_cutoff, put_cutoff=put_cutoff, method=method)
    return res.price, np.asarray(res.status)
