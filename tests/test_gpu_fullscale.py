"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (slow: the sequential oracle takes about a minute per config)."""
import numpy as np
import pytest
import torch

import gen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_cfg3_full_scale_mixed_with_resize():
    """Config 3: 64 batches x 2^20 ops (40/20/40) over U = 2^26 from 1K buckets
    with growth and shrink, then the id-order drain tail; every op's result and
    the expansion trajectory equal the oracle's, batch by batch.

    Mid-round, linear hashing leaves unsplit buckets ~1.35x over-subscribed by
    first-choice keys; the oracle's paper-literal lowest-slot victim rule then
    overflows a 2% stash within the first batches (the GPU's rotating victim
    does not).  Stash capacity does not change any result unless it overflows,
    so the ORACLE runs with a 30% stash while the GPU runs exactly as bench.py
    times it (default 2% stash, batched drains A-29); Pair checks that the GPU
    never dropped an entry (stats.failed == 0)."""
    from gpu_util import Pair
    p = Pair(1024 * 32, oracle_cfg={"stash_fraction": 0.30})
    nbat, bsz, U = 64, 1 << 20, 1 << 26
    for b in range(nbat):
        ops = gen.bernoulli_ops(bsz, 0.4, 0.2, seed=1000 + b)
        ids = gen.uniform_ids(bsz, U, seed=2000 + b)
        p.mixed(ops, gen.keys_of(ids), gen.vals_of(ids))
        sg, so = p.g.stats(), p.o.stats()
        assert (sg["n_buckets"], sg["m"], sg["split"]) == (so["n_buckets"], so["m"], so["split"]), b
        assert sg["count"] == so["count"] and sg["failed"] == 0
    p.check_state()
    assert p.g.stats()["n_buckets"] > 600_000
    for lo in range(0, U, bsz):
        p.erase(gen.keys_of(np.arange(lo, lo + bsz, dtype=np.uint32)))
    sg, so = p.check_state(trajectory=False)
    assert sg["count"] == 0 and (sg["merge_aborts"] > 0 or sg["n_buckets"] == 1024)


def test_cfg4_full_scale_zipf():
    """Config 4: 2^21 buckets (growth off) prefilled with 0.90 * 2^26 keys; Z1 =
    one 2^26-op mixed batch of Zipf(0.99) draws over the present keys (50%
    insert with value = op index, 50% find: 3.3 M copies of the hottest key);
    Z2 = 2^22 Zipf inserts over an absent universe.  Every status / value and
    the final key -> value set equal the oracle's."""
    from gpu_util import Pair
    from phased_model import OP_FIND, OP_INSERT
    nb = 1 << 21
    p = Pair(nb * 32, lf_grow=2.0, lf_shrink=0)
    n_pre = int(0.90 * (1 << 26))
    ids = np.arange(n_pre, dtype=np.uint32)
    p.insert(gen.keys_of(ids), gen.vals_of(ids))
    n1 = 1 << 26
    r1 = gen.zipf_ranks(n1, n_pre, 0.99, seed=7)
    ops = np.where(np.random.default_rng(8).random(n1) < 0.5, OP_INSERT, OP_FIND).astype(np.uint8)
    p.mixed(ops, gen.keys_of((r1 - 1).astype(np.uint32)), np.arange(n1, dtype=np.uint32))
    r2 = gen.zipf_ranks(1 << 22, int(0.05 * (1 << 26)), 0.99, seed=9)
    p.insert(gen.keys_of((r2 - 1 + (1 << 31)).astype(np.uint32)), np.arange(1 << 22, dtype=np.uint32))
    p.check_state()


def test_cfg4_zipf_insert_to_lf_095():
    """Config 4's "90-95% load ... stressing stash fallback" end: 2^21 buckets
    prefilled to LF 0.93, then one batch of 2^23 Zipf(0.99) inserts over an
    absent universe of 0.06 * 2^26 keys (1.39 M distinct, in-batch duplicates
    up to ~4% of the batch per key) lifts the table to LF >= 0.95,
    through Steps 3-4.  Statuses, the final key -> value set and the stash
    contents (seen through finds) equal the oracle's."""
    from gpu_util import Pair
    nb = 1 << 21
    p = Pair(nb * 32, lf_grow=2.0, lf_shrink=0)
    n_pre = int(0.93 * (1 << 26))
    ids = np.arange(n_pre, dtype=np.uint32)
    p.insert(gen.keys_of(ids), gen.vals_of(ids))
    r2 = gen.zipf_ranks(1 << 23, int(0.06 * (1 << 26)), 0.99, seed=9)
    k2 = gen.keys_of((r2 - 1 + (1 << 31)).astype(np.uint32))
    p.insert(k2, np.arange(1 << 23, dtype=np.uint32))
    sg, so = p.check_state()
    assert sg["count"] >= 0.95 * nb * 32, sg["count"] / (nb * 32)
    assert sg["leftovers"] > 0 and sg["evictions"] > 0          # Step 3 ran
    assert sg["stash_pushes"] > 0                               # Step 4 ran
    # every key, including the stashed ones, is found with the oracle's value
    allk = np.concatenate([gen.keys_of(ids[::7]), np.unique(k2)])
    p.find(allk)


def test_cfg2_full_scale_vs_oracle():
    """Config 2 -- the headline bench step -- at full size against the oracle,
    not only its closed form: 2^26 keys into 2,207,529 buckets (LF 0.95, growth
    off) in one batch, then the bench's 2^26 queries (50% hits); every insert
    status, every lookup value / hit and the final key -> value set (sorted
    dumps) are equal.  The oracle alone gets a 30% stash (its paper-literal
    victim overflows 2% in split geometries; stash size changes no result
    unless it overflows), and the GPU must not have dropped an entry."""
    import oracle
    from paper_2510_15095_b200 import HiveTable, u32
    n = 1 << 26
    cap = gen.CFG2_BUCKETS * 32
    t = HiveTable(cap, lf_grow=2.0, lf_shrink=0)
    o = oracle.OracleTable(cap, lf_grow=2.0, lf_shrink=0, stash_fraction=0.30)
    ids = np.arange(n, dtype=np.uint32)
    keys, vals = gen.keys_of(ids), gen.vals_of(ids)
    st = t.insert(u32(keys), u32(vals)).cpu().numpy()
    st_o = o.insert(keys, vals)
    assert (st == st_o).all()
    qids, _ = gen.mixed_queries(n // 2, n // 2, n, seed=202)
    q = gen.keys_of(qids)
    v, f = t.find(u32(q))
    v_o, f_o = o.find(q)
    assert (f.cpu().numpy() == f_o).all()
    assert (v.cpu().numpy().astype(np.uint32) == v_o).all()
    s = t.stats()
    assert s["failed"] == 0 and s["count"] == o.stats()["count"] == n
    kg, vg = t.dump()
    kg, vg = kg.cpu().numpy().astype(np.uint32), vg.cpu().numpy().astype(np.uint32)
    ko, vo = o.dump()
    og, oo = np.argsort(kg, kind="stable"), np.argsort(ko, kind="stable")
    assert (kg[og] == ko[oo]).all() and (vg[og] == vo[oo]).all()
