"""Device-pointer C ABI (fl_price_batch_dev / fl_price_put_bsm /
fl_price_american_call / fl_price_european): torch CUDA tensors
in, torch CUDA tensors out, enqueued on the caller's stream, planned on the
device.  Checked against the reference goldens with the north_star tolerance
(the device derivation uses the CUDA libm, so constants may differ from the
host path's in the last bit)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import NMARG, boundary_check, golden, price_close

pytestmark = pytest.mark.gpu

ERR = {0x100: "ValidationError", 0x200: "StabilityError", 0x300: "DomainError", 0x400: "GeometryError",
       0x500: "NumericalIntegrityError", 0x600: "ValueError"}


def _tensors(g, idx=None):
    import torch

    idx = np.arange(g.n) if idx is None else idx
    f = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a[idx]), dtype=dt, device="cuda")  # noqa: E731
    return (f(g.kind, torch.int8), f(g.S, torch.float64), f(g.K, torch.float64), f(g.R, torch.float64),
            f(g.Y, torch.float64), f(g.V, torch.float64), f(g.E, torch.float64), f(g.T, torch.int64))


def _check(g, idx, price, status, bt=None, bc=None, bn=None):
    bad = []
    for j, i in enumerate(idx):
        ek = str(g.err_kind[i])
        st = int(status[j])
        if ek:
            if ERR.get(st & 0xFF00) != ek:
                bad.append((i, "status", ek, hex(st)))
            continue
        if st != 0:
            bad.append((i, "status", hex(st)))
            continue
        if not price_close(float(price[j]), float(g.price[i]), float(g.K[i])):
            bad.append((i, "price", float(price[j]), float(g.price[i])))
        if bt is not None:
            tr, cr = g.boundary(i)
            c = int(bn[j])
            assert c <= bt.shape[1]
            marg = g.margins(i) if hasattr(g, "bnd_marg") else np.full((len(tr), NMARG), np.nan)
            ok, _, why = boundary_check(int(g.kind[i]), float(g.K[i]), bt[j, :c], bc[j, :c], tr, cr, marg)
            if not ok:
                bad.append((i, "boundary", why))
    assert not bad, bad[:8]


@pytest.mark.parametrize("name", ["edge_fast", "small_fast", "c1_fast", "c2_fast", "c3_fast", "c5_fast"])
def test_dev_entry_matches_goldens(name):
    import torch

    import paper_2303_02317_b200 as fl

    g = golden(name)
    idx = np.arange(g.n)
    k, S, K, R, Y, V, E, T = _tensors(g, idx)
    # fast records are short; options the reference dispatches to its baseline
    # (T <= 2 * cutoff) record every row
    price, status, bt, bc, bn = fl.price_batch_dev(k, S, K, R, Y, V, E, T, bnd_cap=300)
    torch.cuda.synchronize()
    _check(g, idx, price.cpu().numpy(), status.cpu().numpy(), bt.cpu().numpy(), bc.cpu().numpy(),
           bn.cpu().numpy())


@pytest.mark.parametrize("name", ["edge_baseline", "small_baseline"])
def test_dev_entry_baseline_method(name):
    import torch

    import paper_2303_02317_b200 as fl
    from paper_2303_02317_b200 import _native

    g = golden(name)
    idx = np.arange(g.n)
    k, S, K, R, Y, V, E, T = _tensors(g, idx)
    cap = int(g.T.max()) + 2
    price, status, bt, bc, bn = fl.price_batch_dev(k, S, K, R, Y, V, E, T, method=_native.METHOD_BASELINE,
                                                   bnd_cap=cap)
    torch.cuda.synchronize()
    _check(g, idx, price.cpu().numpy(), status.cpu().numpy(), bt.cpu().numpy(), bc.cpu().numpy(),
           bn.cpu().numpy())


def test_dev_per_pricer_entries_on_side_stream():
    """kind_all entries (fl_price_put_bsm / american_call / european), enqueued
    on a non-default stream: results are there once that stream is synced."""
    import torch

    import paper_2303_02317_b200 as fl

    side = torch.cuda.Stream()
    for name, kind in (("c3_fast", 2), ("c2_fast", 1), ("c1_fast", 0)):
        g = golden(name)
        idx = np.arange(0, g.n, 4)
        _, S, K, R, Y, V, E, T = _tensors(g, idx)
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            price, status = fl.price_batch_dev(None, S, K, R, Y, V, E, T, kind_all=kind, max_steps=int(g.T.max()))
        side.synchronize()
        _check(g, idx, price.cpu().numpy(), status.cpu().numpy())


def test_dev_capacity_status():
    """T above max_steps: capacity status (0x707) for the American kinds, the
    European fast path (no workspace) still prices."""
    import torch

    import paper_2303_02317_b200 as fl

    g = golden("c5_fast")
    idx = np.nonzero(g.T >= 4096)[0][::50]
    k, S, K, R, Y, V, E, T = _tensors(g, idx)
    price, status = fl.price_batch_dev(k, S, K, R, Y, V, E, T, max_steps=2048)
    torch.cuda.synchronize()
    st = status.cpu().numpy()
    kinds = g.kind[idx]
    assert np.all(st[kinds != 0] == 0x707)
    assert np.all(st[kinds == 0] == 0)


def test_dev_workspace_query():
    import paper_2303_02317_b200 as fl  # noqa: F401
    from paper_2303_02317_b200 import _native

    a = _native.dev_workspace_bytes(256, 1 << 14)
    b = _native.dev_workspace_bytes(256, 1 << 16)
    assert 0 < a < b
    _native.release_caches()
