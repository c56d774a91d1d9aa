"""The peer-memory exchange of the sharded table on one
GPU: `world` virtual ranks in one process, each with its own Hive table and
exchange buffers, whose phases (route into the owners' inboxes -> owner batch
-> results stored back -> unroute) run in lockstep.  Every rank's results
must equal the oracle's for the union batch in (rank, index) order, which is
the sharded table's contract (sharded.py)."""
import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _run(ranks, kind, per_rank):
    for t, args in zip(ranks, per_rank):
        t.route_phase(kind, *args)
    torch.cuda.synchronize()                      # barrier: every inbox written
    for t in ranks:
        t.serve_phase()
    torch.cuda.synchronize()                      # barrier: every result stored back
    return [t.finish_phase() for t in ranks]


def _split(a, sizes):
    return np.split(a, np.cumsum(sizes)[:-1])


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_p2p_exchange_matches_oracle_on_union_batch(world):
    from paper_2510_15095_b200 import u8, u32
    from paper_2510_15095_b200.sharded import P2PShardedHive
    rng = np.random.default_rng(100 + world)
    region = 6000
    ranks = P2PShardedHive.virtual_group(world, 64 * 32, region, resize_k=16)
    ref = oracle.OracleTable(64 * 32 * world, resize_k=16)
    try:
        for b in range(4):
            # ragged per-rank batches (one rank may be empty), keys shared across
            # ranks so cross-rank duplicates resolve by (rank, index) order
            sizes = [int(x) for x in rng.integers(0, region + 1, world)]
            sizes[b % world] = 0 if b == 2 else sizes[b % world]
            n = sum(sizes)
            keys = rng.integers(0, 6000 * world, n, dtype=np.uint64).astype(np.uint32)
            vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
            ops = gen.bernoulli_ops(n, 0.45, 0.2, seed=b).astype(np.uint8)
            kk, vv, oo = _split(keys, sizes), _split(vals, sizes), _split(ops, sizes)
            got = _run(ranks, "mixed", [(u32(kk[r]), u32(vv[r]), u8(oo[r])) for r in range(world)])
            ev, er = ref.mixed(ops, keys, vals)
            for r, (r8, r32) in enumerate(got):
                assert (r8.cpu().numpy() == _split(er, sizes)[r]).all()
                assert (r32.cpu().numpy().astype(np.uint32) == _split(ev, sizes)[r]).all()
        # single-kind calls over the grown shards
        sizes = [region] * world
        q = rng.integers(0, 8000 * world, region * world, dtype=np.uint64).astype(np.uint32)
        got = _run(ranks, "find", [(u32(x),) for x in _split(q, sizes)])
        fv, ff = ref.find(q)
        for r, (f, v) in enumerate(got):
            assert (f.cpu().numpy() == _split(ff, sizes)[r]).all()
            assert (v.cpu().numpy().astype(np.uint32) == _split(fv, sizes)[r]).all()
        got = _run(ranks, "insert", [(u32(x), u32(x ^ 0x5A5A5A5A)) for x in _split(q, sizes)])
        st = ref.insert(q, q ^ np.uint32(0x5A5A5A5A))
        for r, (s8, _) in enumerate(got):
            assert (s8.cpu().numpy() == _split(st, sizes)[r]).all()
        e = q[::3].copy()
        got = _run(ranks, "erase", [(u32(x),) for x in _split(e, [len(e) // world] * (world - 1) +
                                                             [len(e) - (len(e) // world) * (world - 1)])])
        er = ref.erase(e)
        assert (np.concatenate([g[0].cpu().numpy() for g in got]) == er).all()
        # the shards together hold exactly the oracle's key -> value set
        total = {}
        for t in ranks:
            k, v = t.table.dump()
            total.update(zip(k.cpu().numpy().astype(np.uint32).tolist(), v.cpu().numpy().astype(np.uint32).tolist()))
        assert total == ref.dump_dict()
        assert sum(t.table.stats()["count"] for t in ranks) == ref.stats()["count"]
    finally:
        for t in ranks:
            t.close()


def test_p2p_region_overflow_reports_unsent_ops():
    """A batch larger than its (source, owner) region: the ops past the region
    are not sent (find found = 2, insert status 4), every sent op is exact."""
    from gpu_util import np8, np32
    from paper_2510_15095_b200 import u32
    from paper_2510_15095_b200.sharded import P2PShardedHive
    ranks = P2PShardedHive.virtual_group(1, 64 * 32, 100, lf_grow=2.0, lf_shrink=0)
    try:
        keys = gen.present_keys(130)
        (st, _), = _run(ranks, "insert", [(u32(keys), u32(keys))])
        st = np8(st)
        assert (st[:100] == 0).all() and (st[100:] == 4).all()
        (f, v), = _run(ranks, "find", [(u32(keys),)])
        f, v = np8(f), np32(v)
        assert (f[:100] == 1).all() and (v[:100] == keys[:100]).all() and (f[100:] == 2).all()
    finally:
        for t in ranks:
            t.close()


def test_p2p_lost_peer_poisons_results_without_host_sync():
    """an owner that never answers must not let stale
    results through.  Rank 1 never routes, so rank 0's phase waits time out;
    the unroute kernel sees the timeout marker and reports 6 for every op
    (no host check inside the call), and check() raises and resets it."""
    from gpu_util import np8
    from paper_2510_15095_b200 import HiveError, u32
    from paper_2510_15095_b200.sharded import P2PShardedHive
    ranks = P2PShardedHive.virtual_group(2, 64 * 32, 1000)
    try:
        r0 = ranks[0]
        r0.timeout_ns = 2_000_000                # 2 ms
        r0.route_phase("find", u32(gen.present_keys(500)))
        r0.serve_phase()
        f, _ = r0.finish_phase()
        assert (np8(f) == 6).all()
        with pytest.raises(HiveError):
            r0.check()
        r0.check()                               # the marker was reset
    finally:
        for t in ranks:
            t.close()
