"""Pins of the CPU oracle against things other than itself (paper values,
SPEC worked examples, textbook forms, closed forms, library routines).

Each test names the passage it checks.  See DESIGN.md "Oracle pins".
"""
import numpy as np
import pytest

import oracle
from conftest import ival, read_golden

MASK32 = 0xFFFFFFFF
EMPTY = (1 << 64) - 1


# --- §III-A packed word ----------------------------------------------
def test_pack_unpack_spec_examples():
    n = 0
    for row in read_golden("spec_examples.txt"):
        if row[0] == "pack":
            assert oracle.pack(ival(row[1]), ival(row[2])) == ival(row[3])
            n += 1
        elif row[0] == "unpack":
            assert oracle.unpack(ival(row[1])) == (ival(row[2]), ival(row[3]))
            n += 1
    assert n == 6


def test_pack_roundtrip_and_never_empty():
    rng = np.random.default_rng(1)
    ks = rng.integers(0, MASK32, 20000, dtype=np.uint64)  # excludes 0xFFFFFFFF
    vs = rng.integers(0, MASK32 + 1, 20000, dtype=np.uint64)
    words = set()
    for k, v in zip(ks.tolist(), vs.tolist()):
        w = oracle.pack(k, v)
        assert w != EMPTY
        assert oracle.unpack(w) == (k, v)
        words.add(w)
    assert len(words) == len(set(zip(ks.tolist(), vs.tolist())))  # injective


# --- Listing 1 -------------------------------------------------------
def test_bithash_vectors_from_survey_transcription():
    rows = read_golden("bithash_vectors.txt")
    assert len(rows) == 7
    for k, h1, h2 in rows:
        assert oracle.bithash1(ival(k)) == ival(h1), k
        assert oracle.bithash2(ival(k)) == ival(h2), k


def _wang_hash32shift(key):
    """Thomas Wang's hash32shift in its published alternate form
    ((key << 15) - key - 1 and the 2057 multiply spelt as shifts) — the
    textbook routine Listing 1's BitHash1 is (SURVEY §8(c) pins)."""
    key = ((key << 15) - key - 1) & MASK32
    key = key ^ (key >> 12)
    key = (key + (key << 2)) & MASK32
    key = key ^ (key >> 4)
    key = ((key + (key << 3)) + (key << 11)) & MASK32
    key = key ^ (key >> 16)
    return key


def test_bithash1_is_wang_hash32shift():
    rng = np.random.default_rng(2)
    for k in rng.integers(0, 1 << 32, 20000, dtype=np.uint64).tolist() + [0, 1, MASK32]:
        assert oracle.bithash1(k) == _wang_hash32shift(k)


def _inv_mul(a):
    return pow(a, -1, 1 << 32)


def _inv_xorshr(y, s):
    x = y
    for _ in range(32 // s + 1):
        x = y ^ (x >> s)
    return x & MASK32


def _bithash2_inverse(y):
    """Undo PAPER:242-247 step by step (each step is a bijection of 2^32), so a
    wrong constant, shift or operator in the oracle fails this round trip."""
    y &= MASK32
    # line 247: a = (a ^ 0xb55a4f09) ^ (a >> 16)
    a = _inv_xorshr(y ^ 0xB55A4F09, 16)
    # line 246: a = (a + 0xfd7046c5) + (a << 3)  == 9a + c
    a = ((a - 0xFD7046C5) * _inv_mul(9)) & MASK32
    # line 245: a = (a + 0xd3a2646c) ^ (a << 9) -- solve bit by bit, LSB first
    c, x = 0xD3A2646C, 0
    for i in range(32):
        # bit i of y depends on bits <= i of x
        for bit in (0, 1):
            cand = x | (bit << i)
            lhs = (((cand + c) & MASK32) ^ ((cand << 9) & MASK32))
            if ((lhs >> i) & 1) == ((a >> i) & 1):
                x = cand
                break
    a = x
    # line 244: a = (a + 0x165667b1) + (a << 5)  == 33a + c
    a = ((a - 0x165667B1) * _inv_mul(33)) & MASK32
    # line 243: a = (a ^ 0xc761c23c) ^ (a >> 19)
    a = _inv_xorshr(a ^ 0xC761C23C, 19)
    # line 242: a = (a + 0x7ed55d16) + (a << 12)  == 4097a + c
    a = ((a - 0x7ED55D16) * _inv_mul(4097)) & MASK32
    return a


def test_bithash2_inverts_step_by_step():
    rng = np.random.default_rng(3)
    for k in rng.integers(0, 1 << 32, 3000, dtype=np.uint64).tolist() + [0, 1, MASK32]:
        assert _bithash2_inverse(oracle.bithash2(k)) == k


# --- Linear-hashing address rule (reading A-2) ---------------------
def test_addr_spec_examples():
    rows = [r for r in read_golden("spec_examples.txt") if r[0] == "addr"]
    assert len(rows) == 3
    for _, h, mask, split, b in rows:
        assert oracle.addr(ival(h), ival(mask), ival(split)) == ival(b)


def test_addr_invariants():
    rng = np.random.default_rng(4)
    for _ in range(5000):
        m = int(rng.integers(0, 20))
        mask = (1 << m) - 1
        split = int(rng.integers(0, mask + 2))
        h = int(rng.integers(0, 1 << 32))
        b = oracle.addr(h, mask, split)
        assert b < mask + 1 + split                      # < n_buckets
        if split == 0:
            assert b == h & mask
        # the address is always h mod 2^m or h mod 2^(m+1) (Litwin)
        assert b in (h % (mask + 1), h % (2 * (mask + 1)))


def test_tiny_trace_candidates():
    sizes = {"nb2": (1, 0), "nb3": (1, 1), "nb4": (3, 0), "nb8": (7, 0)}
    rows = read_golden("tiny_trace.txt")
    assert len(rows) == 10
    for row in rows:
        k, h1, h2 = ival(row[0]), ival(row[1]), ival(row[2])
        assert oracle.bithash1(k) == h1 and oracle.bithash2(k) == h2
        for (name, (mask, split)), col in zip(sizes.items(), row[3:]):
            want = tuple(int(x) for x in col.split(","))
            got = (oracle.addr(h1, mask, split), oracle.addr(h2, mask, split))
            assert got == want, (k, name)


def test_alt_bucket_spec_rule():
    # key 0 has candidates (3, 7) at n_b = 8
    assert oracle.alt(0, 3, 7, 0) == 7
    assert oracle.alt(0, 7, 7, 0) == 3
    assert oracle.alt(0, 5, 7, 0) == 3          # neither -> first candidate
    # key 1 has equal candidates (6, 6) at n_b = 8: stays
    assert oracle.alt(1, 6, 7, 0) == 6


# --- lane primitives ------------------------
def test_lane_primitive_spec_examples():
    n = 0
    for row in read_golden("spec_examples.txt"):
        if row[0] == "rank":
            assert oracle.prefix_rank(ival(row[1]), ival(row[2])) == ival(row[3]); n += 1
        elif row[0] == "select":
            assert oracle.select_nth_one(ival(row[1]), ival(row[2])) == ival(row[3]); n += 1
        elif row[0] == "first":
            assert oracle.first_set(ival(row[1])) == ival(row[2]); n += 1
    assert n == 8
    assert oracle.ballot([1, 0, 0, 1] + [0] * 28) == 0b1001
    assert oracle.ballot([0] * 32) == 0 and oracle.ballot([1] * 32) == MASK32


def test_lane_primitives_vs_library_routines():
    rng = np.random.default_rng(5)
    masks = rng.integers(0, 1 << 32, 4000, dtype=np.uint64).tolist() + [0, 1, MASK32, 1 << 31]
    for mask in masks:
        bits = np.array([(mask >> i) & 1 for i in range(32)], np.uint8)
        assert oracle.ballot(bits) == mask
        fs = (mask & -mask).bit_length() - 1                        # library: int ops
        assert oracle.first_set(mask) == fs
        lane = int(rng.integers(0, 32))
        assert oracle.prefix_rank(mask, lane) == (mask & ((1 << lane) - 1)).bit_count()
        ones = np.flatnonzero(bits)                                 # library: numpy
        r = int(rng.integers(0, 33))
        assert oracle.select_nth_one(mask, r) == (int(ones[r]) if r < len(ones) else -1)
        if (mask >> lane) & 1:
            assert oracle.select_nth_one(mask, oracle.prefix_rank(mask, lane)) == lane


# --- split / merge fixtures ------------
def _keys_in(t, b):
    s, fm = t.bucket(b)
    return [int(x) & MASK32 if int(x) != EMPTY else None for x in s], fm


def test_tiny_trace_split_fixture():
    t = oracle.OracleTable(2 * 32, lf_grow=2.0, lf_shrink=0)
    assert (t.insert(np.arange(10), np.arange(10) * 7) == 0).all()
    b0, fm0 = _keys_in(t, 0)
    b1, fm1 = _keys_in(t, 1)
    assert [k for k in b0 if k is not None] == [1, 3, 7, 8, 9]
    assert [k for k in b1 if k is not None] == [0, 2, 4, 5, 6]
    t.expand(1)
    st = t.stats()
    assert (st["n_buckets"], st["m"], st["split"]) == (3, 1, 1)
    b0, fm0 = _keys_in(t, 0)
    b2, fm2 = _keys_in(t, 2)
    assert [k for k in b0 if k is not None] == [3, 7]
    assert b2[:3] == [1, 8, 9] and all(k is None for k in b2[3:])   # compacted, slot order
    assert fm2 == MASK32 & ~0b111
    assert t.check() == ""
    vals, found = t.find(np.arange(10))
    assert found.all() and (vals == np.arange(10) * 7).all()


def _filled(nb, n, seed=0):
    t = oracle.OracleTable(nb * 32, lf_grow=2.0, lf_shrink=0)
    rng = np.random.default_rng(seed)
    keys = rng.choice(1 << 30, n, replace=False).astype(np.uint32)
    assert (t.insert(keys, keys ^ 0x5A5A5A5A) == 0).all()
    return t, keys


def test_spec_expand_examples():
    t, keys = _filled(8, 100)
    t.expand(8)
    st = t.stats()
    assert (st["n_buckets"], st["m"], st["split"]) == (16, 4, 0)
    assert t.check() == ""
    t2, _ = _filled(8, 100)
    t2.expand(2)
    st = t2.stats()
    assert (st["n_buckets"], st["split"]) == (10, 2)
    vals, found = t.find(keys)
    assert found.all() and (vals == keys ^ 0x5A5A5A5A).all()
    # split correctness: every entry is in a candidate under new state
    assert t2.check() == ""


def test_spec_contract_examples():
    t = oracle.OracleTable(8 * 32, lf_grow=2.0, lf_shrink=0)
    keys = np.arange(40, dtype=np.uint32)
    t.insert(keys, keys)
    t.expand(8)
    assert t.stats()["n_buckets"] == 16
    aborted = t.contract(8)
    st = t.stats()
    assert not aborted and (st["n_buckets"], st["m"], st["split"]) == (8, 3, 0)
    vals, found = t.find(keys)
    assert found.all() and (vals == keys).all() and t.check() == ""
    # minimum size: no-op
    t.contract(8)
    assert t.stats()["n_buckets"] == 8


def test_merge_abort_leaves_buckets_identical_and_lowest_free_positions():
    # 2 buckets -> expand to 3 (pair (0,2)), then fill bucket 0 so the merge of
    # (dst 0, src 2) has more movers than free slots.
    t = oracle.OracleTable(2 * 32, lf_grow=2.0, lf_shrink=0)
    t.expand(1)                                                     # n_b = 3
    rng = np.random.default_rng(7)
    cand = rng.choice(1 << 30, 4000, replace=False).astype(np.uint32)
    b1 = np.array([oracle.addr(oracle.bithash1(int(k)), 1, 1) for k in cand])
    b2 = np.array([oracle.addr(oracle.bithash2(int(k)), 1, 1) for k in cand])
    to0 = cand[(b1 == 0) & (b2 == 0)][:30]
    to2 = cand[(b1 == 2) & (b2 == 2)][:5]
    t.insert(to0, to0)
    t.insert(to2, to2)
    before = [t.bucket(b) for b in range(3)]
    assert t.contract(1)                                            # aborts: 5 > 2 free
    after = [t.bucket(b) for b in range(3)]
    for (s0, f0), (s1, f1) in zip(before, after):
        assert (s0 == s1).all() and f0 == f1
    assert t.stats()["n_buckets"] == 3
    # remove 3 from bucket 0 so 5 free slots remain -> merge succeeds and the
    # movers take exactly the 5 lowest free positions
    t.erase(to0[[1, 4, 9]])
    s0, fm0 = t.bucket(0)
    free_pos = [i for i in range(32) if (fm0 >> i) & 1][:5]
    assert not t.contract(1)
    s0b, fm0b = t.bucket(0)
    moved = sorted(int(s0b[i]) & MASK32 for i in free_pos)
    assert moved == sorted(int(k) for k in to2)
    assert t.check() == ""


# --- Step 3 bound (Alg. 3; SPEC acceptance 9) -----------------------------
def test_eviction_cycle_hits_bound_then_stashes():
    for max_ev in (1, 5, 16):
        t = oracle.OracleTable(2 * 32, lf_grow=2.0, lf_shrink=0, max_evictions=max_ev)
        keys = np.arange(100, dtype=np.uint32) * 977 + 13   # > 64 slots: buckets full
        st = t.insert(keys, keys)
        assert (st == 0).all()
        s0 = t.stats()
        assert s0["count"] == 100 and s0["stash_live"] == 100 - 64
        extra = np.array([0xABCDEF], np.uint32)
        assert t.insert(extra, extra)[0] == 0
        s1 = t.stats()
        assert s1["step3_rounds"] - s0["step3_rounds"] == max_ev
        assert s1["lock_acq"] - s0["lock_acq"] == max_ev
        assert s1["step4"] - s0["step4"] == 1
        allk = np.concatenate([keys, extra])
        vals, found = t.find(allk)
        assert found.all() and (vals == allk).all()
        assert t.check() == "" and s1["count"] == 101


# --- shard function ---------------------------------------------------
def test_shard_range_and_uniformity():
    rng = np.random.default_rng(8)
    keys = rng.integers(0, MASK32, 40000, dtype=np.uint64)
    for g in (1, 2, 3, 8):
        s = oracle.shard_array(keys, 0x1234, g)
        assert s.max() < g
        if g > 1:
            counts = np.bincount(s, minlength=g)
            exp = len(keys) / g
            chi2 = ((counts - exp) ** 2 / exp).sum()
            assert chi2 < 30, counts


# --- shard mixer: MurmurHash3 fmix32 -----------------------------------
M32 = 0xFFFFFFFF


def _rotl32(x, r):
    return ((x << r) | (x >> (32 - r))) & M32


def _murmur3_x86_32(data: bytes, seed: int) -> int:
    """MurmurHash3_x86_32 (Appleby) written out block by block; only the final
    avalanche is delegated to the oracle's fmix32, so the published test
    vectors below pin that finaliser (a wrong constant or shift breaks them)."""
    c1, c2 = 0xCC9E2D51, 0x1B873593
    h = seed & M32
    nblocks = len(data) // 4
    for i in range(nblocks):
        k = int.from_bytes(data[4 * i:4 * i + 4], "little")
        k = (k * c1) & M32
        k = _rotl32(k, 15)
        k = (k * c2) & M32
        h ^= k
        h = _rotl32(h, 13)
        h = (h * 5 + 0xE6546B64) & M32
    tail = data[4 * nblocks:]
    k = 0
    if len(tail) >= 3:
        k ^= tail[2] << 16
    if len(tail) >= 2:
        k ^= tail[1] << 8
    if len(tail) >= 1:
        k ^= tail[0]
        k = (k * c1) & M32
        k = _rotl32(k, 15)
        k = (k * c2) & M32
        h ^= k
    h ^= len(data)
    return oracle.fmix32(h)


def test_fmix32_published_murmur3_vectors():
    """Published MurmurHash3_x86_32 vectors: ("", 0) = 0, ("", 1) = 0x514E28B7,
    ("", 0xFFFFFFFF) = 0x81F16F39 -- for the empty message the whole hash IS
    fmix32(seed) -- plus multi-block / tail vectors."""
    assert oracle.fmix32(0) == 0
    assert oracle.fmix32(1) == 0x514E28B7
    assert oracle.fmix32(0xFFFFFFFF) == 0x81F16F39
    assert _murmur3_x86_32(b"", 1) == 0x514E28B7
    assert _murmur3_x86_32(b"abc", 0) == 0xB3DD93FA
    assert _murmur3_x86_32(b"Hello, world!", 0x9747B28C) == 0x24884CBA
    assert _murmur3_x86_32(b"The quick brown fox jumps over the lazy dog", 0x9747B28C) == 0x2FA826CD


def test_fmix32_matches_library_murmur3():
    """Special case reducing to a library routine: scikit-learn's independent
    MurmurHash3_x86_32 of an empty message with seed s is fmix32(s); of a 4-byte
    message it runs one block and then fmix32 (checked through the transcription
    above)."""
    from sklearn.utils import murmurhash3_32
    rng = np.random.default_rng(21)
    for s in rng.integers(0, 1 << 32, 300, dtype=np.uint64).tolist():
        assert oracle.fmix32(s) == murmurhash3_32(b"", seed=s, positive=True)
    for _ in range(200):
        msg = bytes(rng.integers(0, 256, int(rng.integers(0, 12)), dtype=np.uint8).tolist())
        s = int(rng.integers(0, 1 << 32, dtype=np.uint64))
        assert _murmur3_x86_32(msg, s) == murmurhash3_32(msg, seed=s, positive=True)


def _fmix32_inverse(y: int) -> int:
    """fmix32 undone step by step: xorshift-right by 16 is its own inverse on 32
    bits, xorshift by 13 is undone by x ^ x>>13 ^ x>>26, and the multipliers by
    their inverses mod 2^32."""
    y ^= y >> 16
    y = (y * pow(0xC2B2AE35, -1, 1 << 32)) & M32
    y ^= (y >> 13) ^ (y >> 26)
    y = (y * pow(0x85EBCA6B, -1, 1 << 32)) & M32
    y ^= y >> 16
    return y


def test_fmix32_is_a_bijection_with_closed_form_inverse():
    rng = np.random.default_rng(22)
    for y in rng.integers(0, 1 << 32, 3000, dtype=np.uint64).tolist():
        assert oracle.fmix32(_fmix32_inverse(y)) == y


def test_shard_is_multiply_high_not_modulo():
    """shard(k) = (fmix32(k ^ seed) * G) >> 32: keys are built
    through the inverse so that fmix32(k ^ seed) hits chosen values; at G = 3
    the boundary 0x55555555 | 0x55555556 separates the multiply-high rule
    (0 | 1) from `% G` (1 | 2); for G = 2^j the shard is the top j bits."""
    seed = 0x5BD1E995

    def key_for(y):
        return _fmix32_inverse(y) ^ seed
    assert oracle.shard(key_for(0x55555555), seed, 3) == 0
    assert oracle.shard(key_for(0x55555556), seed, 3) == 1
    assert oracle.shard(key_for(0xAAAAAAAA), seed, 3) == 1
    assert oracle.shard(key_for(0xAAAAAAAB), seed, 3) == 2
    assert oracle.shard(key_for(0xFFFFFFFF), seed, 3) == 2
    assert oracle.shard(key_for(0), seed, 5) == 0
    rng = np.random.default_rng(23)
    for y in rng.integers(0, 1 << 32, 2000, dtype=np.uint64).tolist():
        k = key_for(y)
        for j in (1, 2, 3):
            assert oracle.shard(k, seed, 1 << j) == y >> (32 - j)
        assert oracle.shard(k, seed, 1) == 0
        assert oracle.shard(k, seed, 6) == (y * 6) >> 32
