"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the Hive method (no BitHash, no addressing,
no table logic): only the input recipe of DESIGN.md "Input recipe"
(SURVEY §8(d) "Synthetic inputs"):

* key bijection  Key(i) = fmix32(i ^ seed_k) for ids i in [0, 2^32 - 1); the one
  id whose image is the reserved key 0xFFFFFFFF is remapped to
  fmix32(0xFFFFFFFF ^ seed_k) (the image of the never-used id 2^32 - 1), so
  distinct ids always give distinct, valid keys.  Present ids are drawn from
  [0, N); guaranteed-absent ids from [2^31, 2^32 - 1).
* values  Val(i) = fmix32(i ^ seed_v).
* shuffles: numpy PCG64 (``np.random.default_rng(seed)``) permutations.
* Zipf(s) ranks by Hormann-Derflinger rejection-inversion, PCG64 uniforms.
"""
from __future__ import annotations

import numpy as np

SEED_K = 0x9E3779B9
SEED_V = 0x7F4A7C15
INVALID_KEY = 0xFFFFFFFF
ABSENT_BASE = 1 << 31


def fmix32(x: np.ndarray) -> np.ndarray:
    """MurmurHash3 32-bit finaliser (a bijection on uint32)."""
    h = np.asarray(x, dtype=np.uint32).copy()
    with np.errstate(over="ignore"):
        h ^= h >> np.uint32(16)
        h *= np.uint32(0x85EBCA6B)
        h ^= h >> np.uint32(13)
        h *= np.uint32(0xC2B2AE35)
        h ^= h >> np.uint32(16)
    return h


def keys_of(ids, seed: int = SEED_K) -> np.ndarray:
    ids = np.asarray(ids, dtype=np.uint32)
    k = fmix32(ids ^ np.uint32(seed))
    bad = k == np.uint32(INVALID_KEY)
    if bad.any():
        k[bad] = fmix32(np.array([0xFFFFFFFF ^ seed], dtype=np.uint32))[0]
    return k


def vals_of(ids, seed: int = SEED_V) -> np.ndarray:
    return fmix32(np.asarray(ids, dtype=np.uint32) ^ np.uint32(seed))


def present_keys(n: int, seed: int = SEED_K) -> np.ndarray:
    return keys_of(np.arange(n, dtype=np.uint64).astype(np.uint32), seed)


def absent_keys(n: int, seed: int = SEED_K) -> np.ndarray:
    return keys_of((np.arange(n, dtype=np.uint64) + ABSENT_BASE).astype(np.uint32), seed)


def permutation(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).permutation(n)


def mixed_queries(n_hit: int, n_miss: int, n_present: int, seed: int):
    """n_hit ids drawn (without replacement) from [0, n_present) and n_miss
    absent ids, interleaved by a seeded shuffle.  Returns (ids, is_hit)."""
    rng = np.random.default_rng(seed)
    hit_ids = rng.choice(n_present, size=n_hit, replace=False) if n_hit < n_present \
        else rng.permutation(n_present)[:n_hit]
    ids = np.concatenate([hit_ids.astype(np.uint64),
                          np.arange(n_miss, dtype=np.uint64) + ABSENT_BASE])
    is_hit = np.concatenate([np.ones(n_hit, bool), np.zeros(n_miss, bool)])
    p = rng.permutation(len(ids))
    return ids[p].astype(np.uint32), is_hit[p]


def zipf_ranks(n: int, n_elems: int, s: float, seed: int) -> np.ndarray:
    """n draws of Zipf(s) ranks in [1, n_elems] (Hormann & Derflinger 1996,
    rejection-inversion; the Apache Commons formulation)."""
    rng = np.random.default_rng(seed)

    def h_int(x):
        lx = np.log(x)
        t = (1.0 - s) * lx
        helper2 = np.where(np.abs(t) > 1e-8, np.expm1(t) / np.where(t == 0, 1, t), 1 + t / 2)
        return helper2 * lx

    def h_int_inv(x):
        t = x * (1.0 - s)
        t = np.maximum(t, -1.0)
        helper1 = np.where(np.abs(t) > 1e-8, np.log1p(t) / np.where(t == 0, 1, t), 1 - t / 2)
        return np.exp(helper1 * x)

    def h(x):
        return np.exp(-s * np.log(x))

    hx1 = h_int(1.5) - 1.0
    hn = h_int(n_elems + 0.5)
    s_ = 2.0 - h_int_inv(h_int(2.5) - h(2.0))
    out = np.empty(n, dtype=np.int64)
    todo = np.arange(n)
    while len(todo):
        u = hn + rng.random(len(todo)) * (hx1 - hn)
        x = h_int_inv(u)
        k = np.clip(np.floor(x + 0.5), 1, n_elems)
        ok = (k - x <= s_) | (u >= h_int(k + 0.5) - h(k))
        out[todo[ok]] = k[ok].astype(np.int64)
        todo = todo[~ok]
    return out


def bernoulli_ops(n: int, p_insert: float, p_erase: float, seed: int) -> np.ndarray:
    """Opcodes 0 find / 1 insert / 2 erase with the given probabilities."""
    u = np.random.default_rng(seed).random(n)
    op = np.zeros(n, np.uint8)
    op[u < p_insert] = 1
    op[(u >= p_insert) & (u < p_insert + p_erase)] = 2
    return op


def uniform_ids(n: int, universe: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, universe, size=n, dtype=np.uint64).astype(np.uint32)


# --- BASELINE.json configs --------------------------------
CFG2_BUCKETS = 2_207_529          # ceil(2^26 / (0.95 * 32)) buckets -> LF 0.95 at 2^26 keys
CFG1 = dict(capacity=1024 * 32, n_insert=1 << 16, n_find=1 << 16, n_erase=1 << 15)
CFG2 = dict(capacity=CFG2_BUCKETS * 32, n_insert=1 << 26, n_find=1 << 26)
CFG3 = dict(capacity=1024 * 32, batches=64, batch=1 << 20, universe=1 << 26,
            p_insert=0.4, p_erase=0.2)
CFG4 = dict(buckets=1 << 21, prefill_frac=0.90, n_ops=1 << 26, zipf_s=0.99)
