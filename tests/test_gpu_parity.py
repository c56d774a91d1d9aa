"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element, on seeded inputs.  Integer
work: every comparison is bit-exact."""
import numpy as np
import pytest
import torch

import gen
from phased_model import OP_ERASE, OP_FIND, OP_INSERT

pytestmark = pytest.mark.gpu

INVALID = 0xFFFFFFFF


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _pair(capacity, **cfg):
    from gpu_util import Pair
    return Pair(capacity, **cfg)


def test_cfg1_sequence():
    """BASELINE config 1: 2^16 keys into a 1K-bucket table (pre-grow to 3072
    buckets), 2^16 finds (half present), 2^15 erases (half present)."""
    p = _pair(1024 * 32)
    n = 1 << 16
    keys = gen.present_keys(n)
    vals = gen.vals_of(np.arange(n))
    st = p.insert(keys, vals)
    assert (st == 0).all()
    sg, so = p.check_state()
    assert sg["n_buckets"] == 3072
    ids, hit = gen.mixed_queries(n // 2, n // 2, n, seed=101)
    q = gen.keys_of(ids)
    v, f = p.find(q)
    assert (f == hit).all()
    eids, ehit = gen.mixed_queries(n // 4, n // 4, n, seed=102)
    e = p.erase(gen.keys_of(eids))
    assert (e == ehit).all()
    sg, so = p.check_state()
    assert sg["count"] == n - n // 4 and sg["n_buckets"] == 3072    # LF 0.5: no shrink


@pytest.mark.parametrize("n", [0, 1, 7, 31, 33, 1000, 4097])
def test_ragged_batches(n):
    p = _pair(256 * 32, lf_grow=2.0, lf_shrink=0)
    keys = gen.present_keys(n)
    p.insert(keys, gen.vals_of(np.arange(n)))
    q = np.concatenate([keys, gen.absent_keys(n)])
    p.find(q)
    p.erase(keys[: n // 2])
    p.find(q)
    p.check_state()


@pytest.mark.parametrize("n", [0, 1, 7, 33, 4095, 4096, 4097, 3 * 4096 + 5, 1 << 17])
def test_ragged_mixed_batches(n):
    """Mixed batches of every tile shape of the one-pass classification (4096-op
    tiles: empty, partial, exact, one over, several): opcodes 0 / 1 / 2 plus
    invalid opcodes (3, 200: result 0, value 0), repeated keys and the reserved
    key, with growth and shrink on -- results and state equal the oracle's."""
    rng = np.random.default_rng(1000 + n)
    p = _pair(64 * 32, resize_k=16)
    for rnd in range(3):
        ops = rng.choice(np.array([0, 1, 2, 3, 200], np.uint8), size=n, p=[0.3, 0.4, 0.2, 0.05, 0.05])
        ids = rng.integers(0, max(2, n // 2), n, dtype=np.uint64).astype(np.uint32)
        keys = gen.keys_of(ids)
        if n > 10:
            keys[rng.integers(0, n, 3)] = INVALID
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        p.mixed(ops, keys, vals)
        p.check_state()


@pytest.mark.parametrize("n", [1 << 18, (1 << 22) + 4097])
def test_mixed_batches_capture_in_a_cuda_graph(n):
    """With growth and contraction off a PHASED mixed batch never waits on the
    host (classification, elections -- single-table and partitioned with the
    chained sub-table clears -- probes, fix-ups are all stream work), so two
    batches capture into one CUDA graph.  Each replay, with new contents in
    the same input buffers, gives the oracle's results for those batches."""
    import oracle
    from paper_2510_15095_b200 import HiveTable, u8, u32
    cap = -(-n * 2 // 32) * 32 * 2
    g = HiveTable(cap, lf_grow=2.0, lf_shrink=0)
    o = oracle.OracleTable(cap, lf_grow=2.0, lf_shrink=0)
    dev = torch.device("cuda")
    bufs = [(torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.uint32, device=dev),
             torch.empty(n, dtype=torch.uint32, device=dev), torch.empty(n, dtype=torch.uint32, device=dev),
             torch.empty(n, dtype=torch.uint8, device=dev)) for _ in range(2)]
    rng = np.random.default_rng(n)

    def fill():
        host = []
        for ops_t, k_t, v_t, _, _ in bufs:
            ops = rng.choice(np.array([0, 1, 2], np.uint8), size=n, p=[0.4, 0.4, 0.2])
            keys = gen.keys_of(rng.integers(0, n, n, dtype=np.uint64).astype(np.uint32))   # duplicates
            vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
            ops_t.copy_(u8(ops)); k_t.copy_(u32(keys)); v_t.copy_(u32(vals))
            host.append((ops, keys, vals))
        return host

    s = torch.cuda.Stream()
    fill()
    with torch.cuda.stream(s):               # warm-up: sizes every scratch buffer, then reset
        for ops_t, k_t, v_t, vo_t, r_t in bufs:
            g.mixed(ops_t, k_t, v_t, vo_t, r_t, stream=s)
    torch.cuda.synchronize()
    g.clear()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for ops_t, k_t, v_t, vo_t, r_t in bufs:
            g.mixed(ops_t, k_t, v_t, vo_t, r_t, stream=s)
    for rep in range(2):                     # the table carries over between replays
        host = fill()
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        for (ops, keys, vals), (_, _, _, vo_t, r_t) in zip(host, bufs):
            v_o, r_o = o.mixed(ops, keys, vals)
            assert (r_t.cpu().numpy() == r_o).all(), f"replay {rep}: mixed results"
            assert (vo_t.cpu().numpy().astype(np.uint32) == v_o).all(), f"replay {rep}: mixed values"
    assert g.stats()["count"] == o.stats()["count"]
    del graph


def test_duplicates_and_reserved_keys():
    """In-batch duplicates: statuses/erase outputs identical for duplicates
    (present at phase start), value = a member of the accepted set (this
    implementation elects the last op = the oracle's value)."""
    rng = np.random.default_rng(5)
    p = _pair(256 * 32, lf_grow=2.0, lf_shrink=0)
    for it in range(12):
        n = 20000
        keys = rng.integers(0, 3000, n, dtype=np.uint64).astype(np.uint32)
        keys[rng.random(n) < 0.01] = INVALID
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        cand = {}
        for k, v in zip(keys.tolist(), vals.tolist()):
            if k != INVALID:
                cand.setdefault(k, set()).add(v)
        p.insert(keys, vals)
        p.check_state(cand)
        p.find(rng.integers(0, 4000, n, dtype=np.uint64).astype(np.uint32))
        p.erase(rng.integers(0, 4000, n // 4, dtype=np.uint64).astype(np.uint32))
        p.check_state()


def test_high_load_steps_3_and_4():
    """Fill 2^12 buckets to LF 0.97 with growth off: Step 3 and the stash are
    exercised; finds/erases must see stashed keys (A-10, A-11)."""
    nb = 1 << 12
    p = _pair(nb * 32, lf_grow=2.0, lf_shrink=0)
    n = int(0.97 * nb * 32)
    keys = gen.present_keys(n)
    for lo in range(0, n, n // 5 + 1):                        # several batches
        hi = min(n, lo + n // 5 + 1)
        p.insert(keys[lo:hi], gen.vals_of(np.arange(lo, hi)))
    sg, so = p.check_state()
    assert sg["leftovers"] > 0
    q = np.concatenate([keys, gen.absent_keys(10000)])
    p.find(q)
    # re-insert everything (Step 1 replace must reach stashed keys too)
    p.insert(keys, gen.vals_of(np.arange(n)) ^ 0x5555)
    p.find(q)
    p.erase(keys[::3])
    p.find(q)
    p.check_state()


@pytest.mark.parametrize("split", [1, 1536, 4095])
def test_high_load_split_geometry(split):
    """LF 0.97 on a table in the middle of a linear-hashing round (n_b = 2^12 +
    split, so the split-aware eviction victim has split buckets to aim at --
    few, many, all but one): every result, the stash-visible finds and the
    final dump equal the oracle's, and Step 3 did run.  The oracle alone gets
    a 30% stash: its paper-literal lowest-slot victim overflows the 2% stash in
    split states (stash size changes no result unless it overflows; the GPU's
    own stash stays at 2% and must not overflow)."""
    from gpu_util import Pair
    nb = (1 << 12) + split
    p = Pair(nb * 32, oracle_cfg={"stash_fraction": 0.30}, lf_grow=2.0, lf_shrink=0)
    n = int(0.97 * nb * 32)
    keys = gen.present_keys(n)
    for lo in range(0, n, n // 3 + 1):
        hi = min(n, lo + n // 3 + 1)
        p.insert(keys[lo:hi], gen.vals_of(np.arange(lo, hi)))
    sg, so = p.check_state()
    assert sg["n_buckets"] == nb and sg["split"] == split
    assert sg["leftovers"] > 0 and sg["evictions"] > 0
    q = np.concatenate([keys, gen.absent_keys(20000)])
    p.find(q)
    p.erase(keys[1::4])
    p.insert(keys[1::4], gen.vals_of(np.arange(1, n, 4)) ^ 0xA5A5)
    p.find(q)
    p.check_state()


@pytest.mark.parametrize("resize_k", [1024, 7])
def test_mixed_grow_and_shrink(resize_k):
    """BASELINE config 3 shape at small scale: 1K buckets, 40/20/40 mixed
    batches over a universe, growth + contraction; per-batch parity and the
    expansion trajectory (n_b, m, split) equal to the oracle's.

    With small K the unsplit buckets of a linear-hashing round carry about twice
    the load of split ones; the oracle's paper-literal lowest-slot victim rule
    then overflows a 2% stash (1024 of 1311*32 slots at batch 6), so the K=7
    case runs with a 10% stash in both implementations."""
    p = _pair(1024 * 32, resize_k=resize_k, stash_fraction=0.02 if resize_k >= 1024 else 0.10)
    U = 1 << 17
    for b in range(16):
        n = 1 << 14
        ops = gen.bernoulli_ops(n, 0.4, 0.2, seed=1000 + b)
        ids = gen.uniform_ids(n, U, seed=2000 + b)
        p.mixed(ops, gen.keys_of(ids), gen.vals_of(ids ^ b))
        sg, so = p.check_state(trajectory=True)
        assert sg["count"] <= 0.9 * sg["n_buckets"] * 32
    grown = p.g.stats()["n_buckets"]
    assert grown > 1024
    # drain tail: erase the universe in id order -> contraction to the start size
    for lo in range(0, U, 1 << 14):
        ids = np.arange(lo, lo + (1 << 14), dtype=np.uint32)
        p.erase(gen.keys_of(ids))
        sg, so = p.check_state(trajectory=False)                 # merge aborts are layout-dependent
        if sg["merge_aborts"] == 0 and sg["n_buckets"] > 1024:
            assert sg["count"] >= 0.25 * sg["n_buckets"] * 32
    assert p.g.stats()["n_buckets"] < grown and p.g.size() == 0


def test_zipf_contention_at_high_load():
    """BASELINE config 4 shape at small scale: Zipf(0.99) inserts/finds with
    heavy in-batch duplicates on a table near LF 0.95."""
    nb = 1 << 12
    p = _pair(nb * 32, lf_grow=2.0, lf_shrink=0)
    n_pre = int(0.90 * nb * 32)
    keys = gen.present_keys(n_pre)
    p.insert(keys, gen.vals_of(np.arange(n_pre)))
    n = 1 << 16
    r = gen.zipf_ranks(n, n_pre, 0.99, seed=7)
    zk = gen.keys_of((r - 1).astype(np.uint32))
    ops = np.where(np.random.default_rng(8).random(n) < 0.5, OP_INSERT, OP_FIND).astype(np.uint8)
    p.mixed(ops, zk, np.arange(n, dtype=np.uint32))
    # Z2: inserts over an absent universe (LF rises toward 0.95)
    r2 = gen.zipf_ranks(1 << 15, int(0.05 * nb * 32), 0.99, seed=9)
    k2 = gen.keys_of((r2 - 1 + (1 << 31)).astype(np.uint32))
    p.insert(k2, np.arange(len(k2), dtype=np.uint32))
    p.find(np.concatenate([zk[:5000], k2[:5000]]))
    p.check_state()


def test_route_partition_is_stable_and_matches_shard_function():
    import oracle
    from paper_2510_15095_b200 import route, u8, u32, unroute
    from gpu_util import np8
    rng = np.random.default_rng(3)
    for g, n in ((1, 1000), (2, 5000), (8, 100003), (5, 4097)):
        keys = rng.integers(0, INVALID, n, dtype=np.uint64).astype(np.uint32)
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        ops = rng.integers(0, 3, n).astype(np.uint8)
        send_kv, send_ops, pos, counts = route(u32(keys), u32(vals), u8(ops), g, 0xC0FFEE)
        sh = oracle.shard_array(keys, 0xC0FFEE, g)
        assert counts.cpu().numpy().tolist() == np.bincount(sh, minlength=g).tolist()
        order = np.argsort(sh, kind="stable")                    # stable partition
        kv = send_kv.cpu().numpy().view(np.uint64)
        assert (kv == ((vals[order].astype(np.uint64) << 32) | keys[order])).all()
        assert (np8(send_ops) == ops[order]).all()
        p = pos.cpu().numpy()
        assert (p[order] == np.arange(n)).all()
        back, _ = unroute(pos, in8=send_ops)
        assert (np8(back) == ops).all()


def test_cfg2_full_scale_properties():
    """BASELINE config 2 at full size in the bench's launch configuration:
    2^26 unique keys into 2,207,529 buckets (LF 0.95, growth off), then 2^26
    finds with 50% hits.  The expected dictionary is fixed by the inputs
    ({Key(i): Val(i)}), so every output is checked exactly without the oracle."""
    from paper_2510_15095_b200 import HiveTable, u32
    n = 1 << 26
    t = HiveTable(gen.CFG2_BUCKETS * 32, lf_grow=2.0, lf_shrink=0)
    ids = np.arange(n, dtype=np.uint32)
    st = t.insert(u32(gen.keys_of(ids)), u32(gen.vals_of(ids)))
    assert int((st != 0).sum().item()) == 0
    s = t.stats()
    assert s["count"] == n and s["failed"] == 0 and s["n_buckets"] == gen.CFG2_BUCKETS
    qids, hit = gen.mixed_queries(n // 2, n // 2, n, seed=202)
    v, f = t.find(u32(gen.keys_of(qids)))
    f = f.cpu().numpy().astype(bool)
    v = v.cpu().numpy().astype(np.uint32)
    assert (f == hit).all()
    assert (v[hit] == gen.vals_of(qids[hit])).all() and (v[~hit] == 0).all()


def test_partitioned_owner_election_large_batches():
    """Batches large enough for the hash-partitioned election (2^22 ops ->
    2 L2-sized sub-tables) with heavy duplicates: statuses, erase outputs and
    the final dump equal the oracle's."""
    rng = np.random.default_rng(77)
    n = 1 << 22
    p = _pair(-(-(1 << 21) * 100 // (80 * 32)) * 32, lf_grow=2.0, lf_shrink=0)
    keys = rng.integers(0, 1 << 21, n, dtype=np.uint64).astype(np.uint32)
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    p.insert(keys, vals)
    p.check_state()
    p.erase(rng.integers(0, 1 << 22, n, dtype=np.uint64).astype(np.uint32))
    p.check_state()
    p.find(rng.integers(0, 1 << 22, 1 << 20, dtype=np.uint64).astype(np.uint32))


@pytest.mark.parametrize("env", [{}, {"HIVE_ELECT_CHAIN": "0"}, {"HIVE_ELECT_JIT": "0"}, {"HIVE_ELECT_F": "1.2"}])
def test_election_modes_over_many_phases(env):
    """Five rounds of duplicate-heavy 2^22-op partitioned phases (plus small
    single-table phases in between) against the oracle: each part's sub-table
    cleared by the previous part's launch (default), by a memset just before
    it, or all up front; and a denser sub-table (longer probes)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "elect_check.py")],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-3000:]


def test_host_buffer_pipeline_matches_device_path():
    """hive_insert_host / hive_find_host (chunked, multi-stream) give exactly the
    device-buffer results, across several 4 Mi-op chunks and with duplicates."""
    from paper_2510_15095_b200 import HiveTable, u32
    rng = np.random.default_rng(31)
    n = (1 << 22) * 2 + 12345
    keys = rng.integers(0, 1 << 23, n, dtype=np.uint64).astype(np.uint32)
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    q = rng.integers(0, 1 << 24, n, dtype=np.uint64).astype(np.uint32)
    cap = -(-(1 << 23) * 100 // (90 * 32)) * 32
    a = HiveTable(cap, lf_grow=2.0, lf_shrink=0)
    b = HiveTable(cap, lf_grow=2.0, lf_shrink=0)
    st_a = a.insert(u32(keys), u32(vals)).cpu()
    kh = u32(keys, "cpu").pin_memory()
    vh = u32(vals, "cpu").pin_memory()
    qh = u32(q, "cpu").pin_memory()
    st_b = b.insert_host(kh, vh)
    vb, fb = b.find_host(qh)
    torch.cuda.current_stream().synchronize()
    assert torch.equal(st_a, st_b)
    va, fa = a.find(u32(q))
    assert torch.equal(fa.cpu(), fb) and torch.equal(va.cpu(), vb)


def test_overflow_beyond_capacity_and_stash():
    """Degenerate case: a growth-off table of 16 buckets (512 slots, stash
    floor 1024) receives 4096 distinct keys.  Steps 3-4 fill the buckets and
    the stash; every eviction chain that then finds the stash full drops its
    in-hand entry (this op's key or a key it displaced) and marks its op with
    status 3 (include/hive.h); the sticky flag surfaces as HIVE_ESTASHFULL.
    The oracle keeps such entries 'pending' and invisible, so this
    regime is checked by properties, not element parity (A-28):
    one dropped entry per status-3 op, every other key found with its value,
    count = found keys = dump."""
    from paper_2510_15095_b200 import HiveError, HiveTable, u32
    t = HiveTable(16 * 32, max_capacity=16 * 32, lf_grow=2.0, lf_shrink=0)
    n = 4096
    keys = gen.present_keys(n)
    vals = gen.vals_of(np.arange(n))
    st = t.insert(u32(keys), u32(vals)).cpu().numpy()
    assert set(np.unique(st)) <= {0, 3}
    n_bad = int((st == 3).sum())
    assert n_bad == n - (16 * 32 + 1024)                      # every slot and stash entry used
    s = t.stats(allow_failed=True)
    assert s["failed"] == n_bad and s["count"] == n - n_bad
    with pytest.raises(HiveError):
        t.size()
    v, f = t.find(u32(keys))
    v, f = v.cpu().numpy().astype(np.uint32), f.cpu().numpy().astype(bool)
    assert f.sum() == n - n_bad and (v[f] == vals[f]).all()
    dk, dv = t.dump()
    dk, dv = dk.cpu().numpy().astype(np.uint32), dv.cpu().numpy().astype(np.uint32)
    assert len(dk) == n - n_bad and len(set(dk.tolist())) == len(dk)
    assert set(dk.tolist()) == set(keys[f].tolist())


def test_grow_after_regressed_merge_abort():
    """ADVICE r1 (high), reading A-30: a contraction that regresses (m, 0) ->
    (m-1, 2^(m-1)) (A-7) and aborts its first merge leaves the GPU table at
    (m, 0) again; later inserts must still grow it.  Merge aborts depend on the
    slot layout, so seeds are searched until the GPU table hits that case; every
    result and the final key set still equal the oracle's."""
    hit = 0
    for seed in range(400):
        rng = np.random.default_rng(seed)
        p = _pair(64, lf_shrink=0.5, resize_k=2)
        keys = rng.choice(1 << 20, 200, replace=False).astype(np.uint32)
        p.insert(keys[:110], keys[:110])
        er = keys[:110][rng.permutation(110)[: int(rng.integers(50, 100))]]
        p.erase(er)
        sg = p.g.stats()
        if not (sg["merge_aborts"] == 1 and sg["n_buckets"] == 4):
            continue
        assert (sg["m"], sg["split"]) == (2, 0)
        hit += 1
        p.insert(keys[110:], keys[110:])
        sg, so = p.check_state(trajectory=False)
        assert sg["n_buckets"] > 4 and sg["count"] <= 0.9 * sg["n_buckets"] * 32
        p.find(keys)
        if hit >= 3:
            break
    assert hit >= 1


def test_step_breakdown_tool():
    """NEXT-2: the clock64 step breakdown of tools/step_breakdown.py
    on a 2^18-bucket table.  Shares partition the total; Step 4 time appears only
    in batches that stashed; Steps 1-2 dominate at low load; the instrumented
    kernels give the same table as the plain ones (checked against the oracle)."""
    import sys
    sys.path.insert(0, "tools")
    from step_breakdown import breakdown
    rows = breakdown(1 << 18)
    for r in rows:
        assert abs(sum(r["share"]) - 1.0) < 1e-9 and all(c >= 0 for c in r["cycles"])
        assert (r["cycles"][3] > 0) == (r["stashed"] > 0)
        if r["leftovers"] == 0:
            assert r["cycles"][2] == 0
    low = [r for r in rows if r["lf_to"] <= 0.75]
    assert all(r["share"][0] + r["share"][1] > 0.8 for r in low)
    # instrumented insert == plain insert, against the oracle
    p = _pair(1024 * 32, lf_grow=2.0, lf_shrink=0)
    p.g.profile(2)
    keys = gen.present_keys(int(0.96 * 1024 * 32))
    p.insert(keys, gen.vals_of(np.arange(len(keys))))
    p.g.profile(False)
    sg, _ = p.check_state()
    assert sum(sg["step_cycles"]) > 0


@pytest.mark.parametrize("hash_pair", ["bithash", "crc"])
def test_probe_kernels_on_oracle_built_image(hash_pair):
    """hive_load_image: the oracle's own layout -- its
    paper-literal lowest-slot victim rule puts ~1% of the keys in the stash and
    many in their second bucket -- is loaded into the GPU table; the GPU's find /
    erase / insert kernels then run on a layout their insert path never made
    and must match the oracle op by op, split-pointer addressing included
    (2^12 + 1000 buckets; the 3,096 unsplit buckets carry twice the load of
    the split ones, so LF 0.72 fills them to 0.9)."""
    from gpu_util import Pair
    nb = (1 << 12) + 1000
    p = Pair(nb * 32, lf_grow=2.0, lf_shrink=0, hash=hash_pair)
    n = int(0.72 * nb * 32)
    keys = gen.present_keys(n)
    p.o.insert(keys, gen.vals_of(np.arange(n)))
    slots, stash = p.o.image()
    assert len(stash) > 0
    p.g.load_image(torch.from_numpy(slots.view(np.int64)).cuda(), torch.from_numpy(stash.view(np.int64)).cuda())
    assert p.g.stats()["count"] == p.o.stats()["count"]
    q = np.concatenate([keys, gen.absent_keys(20000)])
    p.find(q)
    p.erase(np.concatenate([keys[::5], gen.absent_keys(1000)]))
    p.find(q)
    p.insert(keys[::7], gen.vals_of(np.arange(0, n, 7)) ^ 0xABC)      # replaces, incl. stashed keys
    p.insert(gen.absent_keys(3000), np.arange(3000, dtype=np.uint32))  # new keys into the loaded layout
    p.find(q)
    p.check_state()
