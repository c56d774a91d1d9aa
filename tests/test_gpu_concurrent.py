"""NEXT-4: hive_mixed_concurrent, the whole mixed batch in one cooperative
kernel launch.  Single-type batches must equal the oracle bit-exactly (they
reduce to the PHASED contract); mixed batches must be linearizable per key
(tests/linearizability.py), checked against the GPU table's own dumps before
and after each batch."""
import numpy as np
import pytest
import torch

import gen
from linearizability import check_batch
from phased_model import OP_ERASE, OP_FIND, OP_INSERT

pytestmark = pytest.mark.gpu
INVALID = 0xFFFFFFFF


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _conc(p, ops, keys, vals):
    """One single-type batch through hive_mixed_concurrent vs the oracle."""
    from gpu_util import first_diff, np8, np32
    from paper_2510_15095_b200 import u8, u32
    ops, keys, vals = np.asarray(ops, np.uint8), np.asarray(keys, np.uint32), np.asarray(vals, np.uint32)
    v_g, r_g = p.g.mixed_concurrent(u8(ops), u32(keys), u32(vals))
    v_g, r_g = np32(v_g), np8(r_g)
    v_o, r_o = p.o.mixed(ops, keys, vals)
    p._oracle_ok()
    assert (r_g == r_o).all(), first_diff("result", r_g, r_o, keys)
    assert (v_g == v_o).all(), first_diff("value", v_g, v_o, keys)


def test_single_type_batches_equal_oracle():
    """Insert-only / erase-only / find-only batches with duplicates, reserved
    keys, growth and contraction: bit-exact statuses, values, final dump and
    expansion trajectory."""
    from gpu_util import Pair
    rng = np.random.default_rng(31)
    p = Pair(256 * 32, resize_k=64)
    for it in range(10):
        n = int(rng.integers(1, 40000))
        keys = rng.integers(0, 60000, n, dtype=np.uint64).astype(np.uint32)
        keys[rng.random(n) < 0.01] = INVALID
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        kind = [OP_INSERT, OP_INSERT, OP_ERASE, OP_FIND][it % 4]
        _conc(p, np.full(n, kind, np.uint8), keys, vals)
        p.check_state()
    assert p.g.stats()["grows"] > 0


def test_single_type_insert_high_load_steps_3_4():
    """LF 0.97 with growth off: the eviction / stash stage at the tail of the
    launch; then every key (stashed ones too) through concurrent finds."""
    from gpu_util import Pair
    nb = 1 << 12
    p = Pair(nb * 32, lf_grow=2.0, lf_shrink=0)
    n = int(0.97 * nb * 32)
    keys = gen.present_keys(n)
    for lo in range(0, n, n // 4 + 1):
        hi = min(n, lo + n // 4 + 1)
        _conc(p, np.full(hi - lo, OP_INSERT, np.uint8), keys[lo:hi], gen.vals_of(np.arange(lo, hi)))
    sg, _ = p.check_state()
    assert sg["leftovers"] > 0
    q = np.concatenate([keys, gen.absent_keys(5000)])
    _conc(p, np.zeros(len(q), np.uint8), q, np.zeros(len(q), np.uint32))
    kk = keys[::3]
    _conc(p, np.full(len(kk), OP_ERASE, np.uint8), kk, np.zeros(len(kk), np.uint32))
    p.check_state()


def _dump(t):
    from gpu_util import gpu_dump
    return gpu_dump(t)


@pytest.mark.parametrize("dist", ["uniform", "zipf"])
def test_mixed_batches_are_linearizable(dist):
    """40/20/40 mixed batches over a small key space (many same-key ops per
    batch) and Zipf(0.99) batches: every key's results and final value are
    explained by some order of its insert group, erase group and finds."""
    from gpu_util import np8, np32
    from paper_2510_15095_b200 import HiveTable, u8, u32
    t = HiveTable(512 * 32, resize_k=64)
    rng = np.random.default_rng(7 if dist == "uniform" else 8)
    checked = 0
    for b in range(8):
        n = 1 << 15
        ops = gen.bernoulli_ops(n, 0.4, 0.2, seed=300 + b)
        if dist == "uniform":
            ids = rng.integers(0, 1 << 14, n, dtype=np.uint64).astype(np.uint32)
        else:
            ids = (gen.zipf_ranks(n, 1 << 15, 0.99, seed=400 + b) - 1).astype(np.uint32)
        keys = gen.keys_of(ids)
        keys[rng.random(n) < 0.005] = INVALID
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        ops[rng.random(n) < 0.002] = 7                      # unknown opcode
        before = _dump(t)
        vo, r = t.mixed_concurrent(u8(ops), u32(keys), u32(vals))
        after = _dump(t)
        checked += check_batch(before, ops, keys, vals, np8(r), np32(vo), after)
        s = t.stats()
        assert s["count"] == len(after) and s["failed"] == 0
        assert s["count"] <= 0.9 * s["n_buckets"] * 32 + 1
    assert checked > 10000


def test_mixed_concurrent_large_zipf_batch():
    """cfg4 Z1 shape at reduced size: 2^22 Zipf(0.99) ops (50% insert / 50%
    find) over present keys at LF 0.9: one insert group per key with up to
    ~200 K members; linearizable, and every find of a key that no insert group
    touches returns the prefill value."""
    from gpu_util import np8, np32
    from paper_2510_15095_b200 import HiveTable, u8, u32
    nb = 1 << 16
    t = HiveTable(nb * 32, lf_grow=2.0, lf_shrink=0)
    n_pre = int(0.9 * nb * 32)
    pre = np.arange(n_pre, dtype=np.uint32)
    t.insert(u32(gen.keys_of(pre)), u32(gen.vals_of(pre)))
    n = 1 << 22
    r = gen.zipf_ranks(n, n_pre, 0.99, seed=11)
    keys = gen.keys_of((r - 1).astype(np.uint32))
    ops = np.where(np.random.default_rng(12).random(n) < 0.5, OP_INSERT, OP_FIND).astype(np.uint8)
    vals = np.arange(n, dtype=np.uint32)
    before = _dump(t)
    vo, res = t.mixed_concurrent(u8(ops), u32(keys), u32(vals))
    after = _dump(t)
    check_batch(before, ops, keys, vals, np8(res), np32(vo), after)
    assert (np8(res)[ops == OP_INSERT] == 1).all()          # every key was present
