"""The oracle against brute force (a Python dict under the PHASED contract) and
against the paper's / SPEC's stated behaviour at small scale."""
import numpy as np
import pytest

import gen
import oracle
from phased_model import OP_ERASE, OP_FIND, OP_INSERT, PhasedModel

INVALID = 0xFFFFFFFF


def _random_batch(rng, n, key_space):
    keys = rng.integers(0, key_space, n, dtype=np.uint64).astype(np.uint32)
    keys[rng.random(n) < 0.01] = INVALID                # reserved key
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    return keys, vals


@pytest.mark.parametrize("seed,resize_k,cap", [(11, 4, 64), (12, 1024, 64), (13, 2, 300)])
def test_oracle_vs_dict_phased(seed, resize_k, cap):
    """SPEC acceptance 1 (10^5 ops, key space 2^14), with in-batch duplicates,
    reserved keys, grow and shrink, invariants after every batch."""
    rng = np.random.default_rng(seed)
    t = oracle.OracleTable(cap, lf_grow=0.9, lf_shrink=0.25, resize_k=resize_k)
    m = PhasedModel()
    total = 0
    while total < 100_000:
        n = int(rng.integers(1, 3000))
        kind = rng.choice(["ins", "era", "find", "mixed", "mixed"], p=[0.3, 0.15, 0.1, 0.25, 0.2])
        keys, vals = _random_batch(rng, n, 1 << 14)
        if kind == "ins":
            got = t.insert(keys, vals)
            want, _ = m.insert(keys, vals)
            assert (got == want).all()
        elif kind == "era":
            assert (t.erase(keys) == m.erase(keys)).all()
        elif kind == "find":
            gv, gf = t.find(keys)
            wv, wf = m.find(keys)
            assert (gf == wf).all() and (gv == wv).all()
        else:
            p = rng.dirichlet([1, 1, 1])
            ops = rng.choice([OP_FIND, OP_INSERT, OP_ERASE], n, p=p).astype(np.uint8)
            gv, gr = t.mixed(ops, keys, vals)
            wv, wr, _ = m.mixed(ops, keys, vals)
            assert (gr == wr).all() and (gv == wv).all()
        total += n
        assert t.check() == ""
        assert t.dump_dict() == m.d                       # exact final key->value set
        st = t.stats()
        assert st["count"] == len(m.d)
        assert st["count"] <= 0.9 * st["n_buckets"] * 32 + 1e-9     # LF band (grow)
    # drain tail: erase the whole key space in order, forcing contraction
    for lo in range(0, 1 << 14, 1024):
        ks = np.arange(lo, lo + 1024, dtype=np.uint32)
        assert (t.erase(ks) == m.erase(ks)).all()
        assert t.check() == "" and t.dump_dict() == m.d
        st = t.stats()
        nb_min = max(2, -(-cap // 32))
        if st["n_buckets"] > nb_min and st["merge_aborts"] == 0:
            assert st["count"] >= 0.25 * st["n_buckets"] * 32
    st = t.stats()
    assert st["grows"] > 0 and st["shrinks"] > 0 and st["count"] == 0


def test_fill_to_095_no_failures_small_stash():
    """SPEC acceptance 3: 2^15 buckets, ceil(0.95 * 2^20) distinct keys, growth
    off: zero FailedPending and stash <= 2% of slots."""
    nb = 1 << 15
    n = -(-95 * (nb * 32) // 100)
    t = oracle.OracleTable(nb * 32, lf_grow=2.0, lf_shrink=0)
    keys = gen.present_keys(n)
    st = t.insert(keys, gen.vals_of(np.arange(n)))
    assert (st == 0).all() and t.rc == 0
    s = t.stats()
    assert s["pending"] == 0 and s["count"] == n
    assert s["stash_live"] <= 0.02 * nb * 32
    # ~1% of slots stashed with the paper's victim rule
    assert 0.002 < s["stash_live"] / (nb * 32) < 0.02
    assert s["max_depth"] <= 16
    assert t.check() == ""
    vals, found = t.find(keys)
    assert found.all() and (vals == gen.vals_of(np.arange(n))).all()


def test_step_distribution_at_075():
    """SPEC acceptance 4 / PAPER:636: at LF 0.75, Step-3 entries
    <= 5% and lock acquisitions <= 2% of inserts (count-based, loose)."""
    nb = 1 << 14
    n = int(0.75 * nb * 32)
    t = oracle.OracleTable(nb * 32, lf_grow=2.0, lf_shrink=0)
    t.insert(gen.present_keys(n), gen.vals_of(np.arange(n)))
    s = t.stats()
    assert s["step3_entries"] <= 0.05 * n
    assert s["lock_acq"] <= 0.02 * n
    assert s["step1"] + s["step2"] + s["step3_ok"] + s["step4"] == n
    # most keys sit in their first bucket under first-fit (99.4%)
    assert s["in_b1"] / n > 0.98


def test_resize_round_trip():
    """SPEC acceptance 5: fill past 0.9 (expansions), erase below 0.25
    (contractions); key multiset preserved; size returns to the start."""
    t = oracle.OracleTable(16 * 32, lf_grow=0.9, lf_shrink=0.25, resize_k=8)
    ids = np.arange(4000)
    keys = gen.present_keys(4000)
    t.insert(keys, gen.vals_of(ids))
    s = t.stats()
    assert s["n_buckets"] > 16 and s["count"] <= 0.9 * s["n_buckets"] * 32
    vals, found = t.find(keys)
    assert found.all() and (vals == gen.vals_of(ids)).all()
    t.erase(keys[:3990])
    s = t.stats()
    vals, found = t.find(keys[3990:])
    assert found.all() and (vals == gen.vals_of(ids[3990:])).all()
    assert s["n_buckets"] == 16 and t.check() == ""


def test_n_zero_and_reserved_key():
    t = oracle.OracleTable(64)
    e = np.zeros(0, np.uint32)
    assert len(t.insert(e, e)) == 0 and len(t.erase(e)) == 0
    st = t.insert([INVALID, 5], [1, 2])
    assert st.tolist() == [2, 0]
    v, f = t.find([INVALID, 5])
    assert f.tolist() == [0, 1] and v[1] == 2
    assert t.erase([INVALID]).tolist() == [0]


def test_phased_duplicates_example():
    """Duplicates: every duplicate reports present(k) at its phase start; the
    oracle keeps the last written value (one member of the accepted set)."""
    t = oracle.OracleTable(64, lf_grow=2.0, lf_shrink=0)
    t.insert([7], [70])
    st = t.insert([7, 8, 8, 7], [71, 80, 81, 72])
    assert st.tolist() == [1, 0, 0, 1]
    v, f = t.find([7, 8])
    assert v.tolist() == [72, 81]
    ops = [OP_INSERT, OP_ERASE, OP_FIND, OP_ERASE, OP_INSERT]
    vo, r = t.mixed(ops, [9, 8, 8, 8, 9], [90, 0, 0, 0, 91])
    # insert phase: 9 new (status 0 twice); erase phase: 8 present at start (1, 1);
    # find phase runs after erase: 8 absent.
    assert r.tolist() == [0, 1, 0, 1, 0]
    v, f = t.find([9])
    assert v.tolist() == [91]


def test_cfg1_expansion_trajectory_closed_form():
    """SURVEY §8(d) cfg1 (BASELINE configs[0]): 1024 buckets, lf 0.9 / 0.25, K = 1024.
    Growing before the 2^16-key insert phase while (count + n_ins) > 0.9 * n_b * 32
    (reading A-19) in K-bucket batches: 29,491 < 65,536 ->
    1024 -> 2048 buckets (one whole round: m = 11, split = 0), 58,982 < 65,536 ->
    3072 (m = 11, split = 1024), 88,474 >= 65,536 stop; LF 2/3.  2^15 erases
    (half present) leave 49,152 keys = LF 0.5 > 0.25: no contraction."""
    t = oracle.OracleTable(1024 * 32, lf_grow=0.9, lf_shrink=0.25, resize_k=1024)
    n = 1 << 16
    ids = np.arange(n, dtype=np.uint32)
    st = t.insert(gen.keys_of(ids), gen.vals_of(ids))
    assert (st == 0).all()
    s = t.stats()
    assert (s["n_buckets"], s["m"], s["split"], s["grows"], s["count"]) == (3072, 11, 1024, 2, n)
    qids, hit = gen.mixed_queries(n // 2, n // 2, n, seed=101)
    vals, found = t.find(gen.keys_of(qids))
    assert (found == hit).all() and (vals[hit == 1] == gen.vals_of(qids[hit == 1])).all()
    eids = np.concatenate([np.arange(n // 4, dtype=np.uint32), qids[hit == 0][: n // 4]])
    er = t.erase(gen.keys_of(eids))
    assert er.sum() == n // 4
    s = t.stats()
    assert (s["n_buckets"], s["count"], s["shrinks"]) == (3072, 49_152, 0)
    assert t.check() == ""


def test_grow_after_regressed_merge_abort():
    """ADVICE r1 (high) regression, reading A-30: a contraction that regresses
    (m, 0) -> (m-1, 2^(m-1)) (A-7) and then aborts its first merge must leave a
    state the expansion can continue from.  Before the fix the table stayed at
    4 buckets with 141 keys (LF 1.1) because ExpandBatch saw split == 2^m."""
    rng = np.random.default_rng(64)
    t = oracle.OracleTable(64, lf_grow=0.9, lf_shrink=0.5, resize_k=2)
    keys = rng.choice(1 << 20, 200, replace=False).astype(np.uint32)
    t.insert(keys[:110], keys[:110])
    assert (t.stats()["n_buckets"], t.stats()["m"], t.stats()["split"]) == (4, 2, 0)
    er = keys[:110][rng.permutation(110)[: int(rng.integers(50, 100))]]
    t.erase(er)
    s = t.stats()
    assert s["merge_aborts"] == 1 and s["n_buckets"] == 4      # the first merge aborted
    assert s["split"] < (1 << s["m"])                          # normalised state (A-30)
    t.insert(keys[110:], keys[110:])
    s = t.stats()
    assert s["count"] <= 0.9 * s["n_buckets"] * 32 and s["n_buckets"] > 4
    assert t.check() == ""
