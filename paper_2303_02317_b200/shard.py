"""Option-batch sharding across GPUs: every option is
independent, so each rank prices its own subset and results are only
gathered -- no collective sits on the data path.

* ``option_cost``: the survey's cost model (put ~24.8 T log2^2 T, American call
  ~10 T log2^2 T, European ~c_e T);
* ``lpt_shards``: longest-processing-time greedy partition of a batch;
* ``gather_prices``: rank-0 assembly of the per-rank results (outside any
  timed region) through ``torch.distributed`` (gloo on CPU, nccl on GPUs).
Per-option arithmetic never depends on the shard, so results are identical
at any rank count.
"""

from __future__ import annotations

import numpy as np

__all__ = ["option_cost", "lpt_shards", "gather_prices"]

_C_PUT, _C_CALL, _C_EURO = 24.8, 10.0, 8.0


def option_cost(kind, T) -> np.ndarray:
    """Estimated work per option (arbitrary units, comparable across kinds)."""
    kind = np.asarray(kind)
    T = np.asarray(T, dtype=np.float64)
    l2 = np.maximum(np.log2(np.maximum(T, 2.0)), 1.0)
    dac = np.where(kind == 2, _C_PUT, _C_CALL) * T * l2 * l2
    return np.where(kind == 0, _C_EURO * T, dac)


def lpt_shards(kind, T, nshard: int) -> list[np.ndarray]:
    """Cost-balanced partition: options sorted by decreasing cost, each given
    to the least-loaded shard.  Returns the sorted index array of each shard."""
    if nshard < 1:
        raise ValueError("nshard must be >= 1")
    c = option_cost(kind, T)
    order = np.argsort(-c, kind="stable")
    load = np.zeros(nshard)
    owner = np.empty(len(c), dtype=np.int64)
    for i in order:
        r = int(np.argmin(load))
        owner[i] = r
        load[r] += c[i]
    return [np.nonzero(owner == r)[0] for r in range(nshard)]


def gather_prices(local_idx: np.ndarray, price: np.ndarray, status: np.ndarray, total: int, dist, rank: int):
    """Assemble (price[total], status[total]) on rank 0 from every rank's
    (indices, price, status); other ranks get (None, None)."""
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (np.asarray(local_idx), np.asarray(price), np.asarray(status)))
    if rank != 0:
        return None, None
    P = np.full(total, np.nan)
    St = np.full(total, -1, dtype=np.int32)
    for idx, p, s in parts:
        P[idx] = p
        St[idx] = s
    return P, St
