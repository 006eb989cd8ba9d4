"""Determinism contract (SURVEY 7 hard part 4, 8(e)): an option's price and
boundary records are bit-identical regardless of the batch it is priced in
and of the shard that prices it.  The persistent kernels hand options to
chains from a global queue, FFT groups steal tasks and chains share CTAs, so
this is checked, not argued: the same options are priced

* alone (one option per launch),
* inside the 256-option headline batch,
* inside a C5-style mix of all three kinds and every T,
* inside each LPT shard of a 4-way split of that mix (shard.lpt_shards),
* through both dispatches of a mixed batch (one mixed kernel / put then call kernel),
* and through the multi-device entry on the one visible device,

and every result must be identical to the bit."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _price(kind, S, K, R, Y, V, E, T):
    from paper_2303_02317_b200 import _native

    return _native.price_batch_full(np.asarray(kind, np.int8), S, K, R, Y, V, E, np.asarray(T, np.int64),
                                    lam=0.4, method=0, bnd_cap=128)


def _fields(g, idx):
    return [getattr(g, f)[idx] for f in ("kind", "S", "K", "R", "Y", "V", "E", "T")]


def _same(res_a, ia, res_b, ib):
    if res_a.status[ia] != res_b.status[ib]:
        return False
    if res_a.price[ia].tobytes() != res_b.price[ib].tobytes():
        return False
    ta, ca = res_a.boundary(ia)
    tb, cb = res_b.boundary(ib)
    return np.array_equal(ta, tb) and np.array_equal(ca, cb)


def test_headline_batch_vs_alone():
    g = golden("c6_fast")
    full = _price(*_fields(g, np.arange(g.n)))
    probe = [0, 1, 17, 100, 200, 255]
    for i in probe:
        one = _price(*_fields(g, np.array([i])))
        assert _same(full, i, one, 0), i
    # a different composition: the probes reversed, interleaved with C3 options
    c3 = golden("c3_fast")
    kinds, cols = [], []
    for i in reversed(probe):
        kinds.append((g, i))
        kinds.append((c3, i))
    f = [np.array([getattr(src, name)[i] for src, i in kinds]) for name in ("kind", "S", "K", "R", "Y", "V", "E", "T")]
    mix = _price(*f)
    for pos, i in enumerate(reversed(probe)):
        assert _same(full, i, mix, 2 * pos), i


def test_mix_and_lpt_shards():
    from paper_2303_02317_b200 import shard

    g5 = golden("c5_fast")
    # a C5-style mix: every stratum of the golden sample, shuffled
    rng = np.random.default_rng(5)
    idx = rng.permutation(g5.n)[:600]
    f = _fields(g5, idx)
    whole = _price(*f)
    for nshard in (4,):
        for part in shard.lpt_shards(f[0], f[7], nshard):
            sub = _price(*[a[part] for a in f])
            for j, i in enumerate(part):
                assert _same(whole, int(i), sub, j), (nshard, int(i))
    # the same options inside the headline batch composition: puts at 2^16 first
    g6 = golden("c6_fast")
    head = _fields(g6, np.arange(64))
    both = [np.concatenate([a, b]) for a, b in zip(head, f)]
    res = _price(*both)
    for j in range(len(idx)):
        assert _same(whole, j, res, 64 + j), j


def test_mixed_batch_dispatch_is_bit_identical(monkeypatch):
    """A mixed put / call batch runs either in the one mixed kernel or as the put
    kernel then the call kernel (fl_abi.cu picks by the per-kind fill ratio;
    FL_SPLIT_KINDS forces either): both dispatches give the same bits, and both
    match the golden prices."""
    from conftest import price_close

    g5 = golden("c5_fast")
    rng = np.random.default_rng(55)
    idx = rng.permutation(g5.n)[:400]
    f = _fields(g5, idx)
    assert (f[0] == 1).any() and (f[0] == 2).any()
    monkeypatch.setenv("FL_SPLIT_KINDS", "0")
    mixed = _price(*f)
    monkeypatch.setenv("FL_SPLIT_KINDS", "1")
    split = _price(*f)
    monkeypatch.delenv("FL_SPLIT_KINDS")
    auto = _price(*f)
    for j, i in enumerate(idx):
        assert _same(mixed, j, split, j), int(i)
        assert _same(mixed, j, auto, j), int(i)
        if np.isfinite(g5.price[i]):
            assert price_close(split.price[j], g5.price[i], g5.K[i]), int(i)


def test_multi_device_entry_matches_single():
    """price_batch_multi on devices=[0] is bit-identical to price_batch."""
    import paper_2303_02317_b200 as fl
    from paper_2303_02317_b200 import _native

    g5 = golden("c5_fast")
    idx = np.arange(0, g5.n, 3)
    f = _fields(g5, idx)
    ref = _native.price_batch(*f, lam=0.4)
    p, st = fl.price_batch_multi(*f, devices=[0])
    assert np.array_equal(st, ref.status)
    assert p.tobytes() == ref.price.tobytes()


@pytest.mark.parametrize("kind,T", [(2, 4096), (2, 777), (1, 4096), (1, 1500), (0, 3000)])
def test_sweep_cluster_vs_per_cta(kind, T):
    """O(T^2) baselines: one option alone runs on a cluster of SMs
    (put_sweep_cluster_kernel / call_sweep_cluster_kernel, DSMEM halos);
    the same option inside a 160-option batch runs on one CTA.  Price and
    every boundary record must agree to the bit."""
    from paper_2303_02317_b200 import _native

    n = 160
    rng = np.random.default_rng(kind * 100 + T)
    S = np.full(n, 100.0) if kind == 2 else rng.uniform(80, 120, n)
    K = np.full(n, 100.0)
    R = np.full(n, 0.05)
    Y = np.full(n, 0.0 if kind == 2 else 0.03)
    V = rng.uniform(0.2, 0.4, n)
    E = np.full(n, 365.0)
    ks, Ts = np.full(n, kind, np.int8), np.full(n, T, np.int64)

    def run(sel):
        return _native.price_batch_full(ks[sel], S[sel], K[sel], R[sel], Y[sel], V[sel], E[sel], Ts[sel],
                                        lam=0.4, method=_native.METHOD_BASELINE, bnd_cap=T + 2)

    batch = run(np.arange(n))
    assert np.all(batch.status == 0)
    for i in (0, 77):
        one = run(np.array([i]))
        assert one.status[0] == 0
        assert _same(batch, i, one, 0), (kind, T, i)
        if kind == 1:
            assert len(one.boundary(0)[0]) == T + 1
