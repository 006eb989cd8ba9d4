"""Multi-rank host logic on CPU (gloo, world_size 2): each rank takes its LPT
shard of a C5-style batch, "prices" it (a deterministic per-option stand-in:
the work itself needs a GPU), and rank 0 reassembles the batch through
shard.gather_prices -- the same code bench.py runs over NCCL.  Checks that the
shards partition the batch, are cost-balanced, and that per-option results do
not depend on the rank count."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2303_02317_b200.shard import gather_prices, lpt_shards, option_cost
    from paper_2303_02317_b200.workloads import draw_config

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = draw_config(5, n=600)
    idx = lpt_shards(b.kind, b.T, world)[rank]
    # the library's own plan (fl_shard_plan, used by fl_price_batch_multi)
    # gives every rank the same shard
    from paper_2303_02317_b200._native import shard_plan

    assert np.array_equal(np.nonzero(shard_plan(b.kind, b.T, world) == rank)[0], idx)
    local = b.subset(idx)
    # stand-in for the per-option price: a function of the option alone
    price = local.S * 1e-3 + local.K + np.log2(local.T)
    status = np.zeros(len(local), dtype=np.int32)
    load = np.array([option_cost(local.kind, local.T).sum()])
    loads = [None] * world
    dist.all_gather_object(loads, float(load[0]))
    P, St = gather_prices(idx, price, status, len(b), dist, rank)
    if rank == 0:
        np.savez(out_path, P=P, St=St, loads=np.asarray(loads))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shard_and_gather(tmp_path):
    sys.path.insert(0, ROOT)
    from paper_2303_02317_b200.workloads import draw_config

    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    z = np.load(out)
    b = draw_config(5, n=600)
    expect = b.S * 1e-3 + b.K + np.log2(b.T)
    assert np.array_equal(z["P"], expect)  # every option exactly once, shard-independent
    assert np.all(z["St"] == 0)
    loads = z["loads"]
    assert loads.max() <= 1.05 * loads.mean()
