"""GPU parity for the hash study: the device hash
functions (BitHash1/2 from Listing 1, the constant-memory CRC-32 / CRC-64
pair of §V-B) bit-exact against the oracle, the collision count Y of
Theorem 1 exact, and a Hive table built on the CRC pair equal to the oracle
table built on the same pair."""
import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu

FNS = {"bithash1": oracle.bithash1, "bithash2": oracle.bithash2, "crc32": oracle.crc32,
       "crc64": oracle.crc64_lo}


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _dev(a):
    from paper_2510_15095_b200 import u32
    return u32(np.asarray(a, np.uint32))


@pytest.mark.parametrize("fn", list(FNS))
def test_hash_functions_bit_exact(fn):
    from paper_2510_15095_b200 import hive
    edge = [0, 1, 2, 0xFF, 0x100, 0xFFFF, 0x10000, 0x7FFFFFFF, 0x80000000, 0xFFFFFFFE, 0xFFFFFFFF]
    keys = np.concatenate([np.array(edge, np.uint32),
                           np.random.default_rng(5).integers(0, 1 << 32, 20000, dtype=np.uint64).astype(np.uint32)])
    h = hive.hash_keys(fn, _dev(keys)).cpu().numpy().astype(np.uint32)
    exp = np.array([FNS[fn](int(k)) for k in keys], np.uint32)
    assert (h == exp).all()
    # full-size launch (2^24 keys, many grid-stride rounds): sampled check
    big = gen.present_keys(1 << 24)
    hb = hive.hash_keys(fn, _dev(big)).cpu().numpy().astype(np.uint32)
    idx = np.random.default_rng(6).integers(0, len(big), 4096)
    assert all(int(hb[i]) == FNS[fn](int(big[i])) for i in idx)
    assert (hive.hash_keys(fn, _dev(np.zeros(0, np.uint32))).numel() == 0)


@pytest.mark.parametrize("fn", list(FNS))
def test_collision_count_exact(fn):
    """Y = sum_b (L_b - 1)_+ (Theorem 1) from the device bitmap equals the
    oracle's histogram, for power-of-two and odd bin counts."""
    from paper_2510_15095_b200 import hive
    for n in (0, 512, 1 << 16, 1 << 20):
        keys = gen.present_keys(n) if n else np.zeros(0, np.uint32)
        for m in (512 * 512, 1000003, 33):
            assert hive.collisions(fn, _dev(keys), m) == oracle.observed_collisions(fn, keys, m), (n, m)


def _pair(capacity, **cfg):
    from gpu_util import Pair
    return Pair(capacity, hash="crc", **cfg)


def test_crc_pair_table_cfg1_sequence():
    """The CRC-32 / CRC-64 pair (HIVE_HASH_CRC) through insert (growing from
    1K buckets), find and erase, element by element against the oracle on the
    same pair, final layout trajectory included."""
    p = _pair(1024 * 32)
    n = 1 << 16
    keys = gen.present_keys(n)
    assert (p.insert(keys, gen.vals_of(np.arange(n))) == 0).all()
    p.check_state()
    ids, hit = gen.mixed_queries(n // 2, n // 2, n, seed=101)
    v, f = p.find(gen.keys_of(ids))
    assert (f == hit).all()
    eids, ehit = gen.mixed_queries(n // 4, n // 4, n, seed=102)
    assert (p.erase(gen.keys_of(eids)) == ehit).all()
    p.check_state()


def test_crc_pair_high_load_and_mixed_resize():
    """Steps 3-4 at LF 0.97 (growth off), then 40/20/40 mixed batches with
    growth and contraction — both on the CRC pair."""
    nb = 1 << 12
    p = _pair(nb * 32, lf_grow=2.0, lf_shrink=0)
    n = int(0.97 * nb * 32)
    keys = gen.present_keys(n)
    for lo in range(0, n, n // 5 + 1):
        hi = min(n, lo + n // 5 + 1)
        p.insert(keys[lo:hi], gen.vals_of(np.arange(lo, hi)))
    sg, _ = p.check_state()
    assert sg["leftovers"] > 0
    p.find(np.concatenate([keys, gen.absent_keys(10000)]))
    p.erase(keys[::3])
    p.find(keys)
    p.check_state()

    q = _pair(1024 * 32)
    U = 1 << 17
    for b in range(8):
        m = 1 << 14
        ops = gen.bernoulli_ops(m, 0.4, 0.2, seed=3000 + b)
        ids = gen.uniform_ids(m, U, seed=4000 + b)
        q.mixed(ops, gen.keys_of(ids), gen.vals_of(ids ^ b))
        q.check_state(trajectory=True)
    assert q.g.stats()["n_buckets"] > 1024


def test_crc_pair_decides_placement():
    """Decisive layout check: 100 keys sharing one (CRC-32, CRC-64) candidate
    pair in a 64-bucket table fill both buckets and push 36 to the stash on the
    CRC table (as in the oracle), while the BitHash table spreads them."""
    from paper_2510_15095_b200 import HiveTable
    nb = 64
    pool = gen.present_keys(1 << 20)
    c = {}
    for k in pool.tolist():
        pr = (oracle.crc32(k) & (nb - 1), oracle.crc64_lo(k) & (nb - 1))
        if pr[0] != pr[1]:
            c.setdefault(pr, []).append(k)
    keys = np.array(max(c.values(), key=len)[:100], np.uint32)
    assert len(keys) == 100
    p = _pair(nb * 32, lf_grow=2.0, lf_shrink=0, stash_fraction=0.5)
    p.insert(keys, gen.vals_of(np.arange(100)))
    p.find(keys)
    sg, so = p.check_state()
    assert sg["stash_used"] == so["stash_live"] == 36
    assert sg["in_b1"] == 32                       # b1 full, b2 full, 36 stashed
    t = HiveTable(nb * 32, lf_grow=2.0, lf_shrink=0, stash_fraction=0.5)
    t.insert(_dev(keys), _dev(gen.vals_of(np.arange(100))))
    assert t.stats()["stash_used"] == 0


@pytest.mark.parametrize("n,n_blocks", [(1, 1), (1000, 3), (33333, 4097), (1 << 20, 1 << 16)])
def test_gather_ceiling_reads_the_named_blocks(n, n_blocks):
    """hive_gather_ceiling (SURVEY §8(d) calibration ceiling, not the method):
    out[i] = xor of the 64 32-bit words of block (fmix32(k_i) * n_blocks) >> 32."""
    from paper_2510_15095_b200 import hive
    rng = np.random.default_rng(n + n_blocks)
    blocks = rng.integers(0, 1 << 63, n_blocks * 32, dtype=np.int64)
    keys = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    out = hive.gather_ceiling(torch.from_numpy(blocks).cuda(), _dev(keys)).cpu().numpy().astype(np.uint32)
    b = (gen.fmix32(keys).astype(np.uint64) * np.uint64(n_blocks)) >> np.uint64(32)
    words = blocks.view(np.uint32).reshape(n_blocks, 64)
    exp = np.bitwise_xor.reduce(words[b.astype(np.int64)], axis=1)
    assert (out == exp).all()


def test_gather_ceiling_rw_store_and_cas():
    """hive_gather_ceiling_rw: mode 1 stores word0 ^ 1 into slot (k & 31) of
    the key's block; mode 2 CASes that slot from word0 to word0 ^ 1 (so only
    slot 0, or a slot equal to word0, changes).  Keys here hit distinct blocks."""
    from paper_2510_15095_b200 import hive
    rng = np.random.default_rng(11)
    n_blocks = 1 << 16
    keys = rng.integers(0, 1 << 32, 3000, dtype=np.uint64).astype(np.uint32)
    b = ((gen.fmix32(keys).astype(np.uint64) * np.uint64(n_blocks)) >> np.uint64(32)).astype(np.int64)
    _, first = np.unique(b, return_index=True)
    keys, b = keys[np.sort(first)], b[np.sort(first)]            # one key per block
    orig = rng.integers(0, 1 << 63, n_blocks * 32, dtype=np.int64)
    for mode in (1, 2):
        dev = torch.from_numpy(orig.copy()).cuda()
        hive.gather_ceiling_rw(dev, _dev(keys), mode)
        got = dev.cpu().numpy().reshape(n_blocks, 32)
        exp = orig.copy().reshape(n_blocks, 32)
        j = (keys & 31).astype(np.int64)
        if mode == 1:
            exp[b, j] = exp[b, 0] ^ 1
        else:
            hit = exp[b, j] == exp[b, 0]
            exp[b[hit], j[hit]] = exp[b[hit], 0] ^ 1
        assert (got == exp).all(), mode
