"""CPU oracle for the Hive hash table — TEST INFRASTRUCTURE ONLY.

A plain sequential implementation of arXiv 2510.15095 (reference PAPER.md),
written in C++ (``hive_oracle.cpp``) and loaded here with ctypes.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2510_15095_b200`` never imports it and shares no code with it.

Parity status: see DESIGN.md "Oracle pins".  Slot placement, stash
membership and eviction counts are not observable and are "parity unpinned"
by design (checked by invariants only).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hive_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

OP_FIND, OP_INSERT, OP_ERASE = 0, 1, 2
INVALID_KEY = 0xFFFFFFFF


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (plain -O2, no parallelism)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "hive_oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class _Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64 if n not in ("m", "split") else ctypes.c_uint32) for n in (
        "n_buckets", "m", "split", "count", "stash_live", "stash_cap", "step1", "step2",
        "step3_entries", "step3_ok", "step3_rounds", "step4", "lock_acq", "max_depth", "grows",
        "shrinks", "merge_aborts", "pending", "in_b1")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u32, u64, f32, vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_float, ctypes.c_void_p
        L.oracle_create.restype = vp
        L.oracle_create.argtypes = [u64, u64, f32, f32, u32, u32, f32]
        L.oracle_destroy.argtypes = [vp]
        for name, args in {
            "oracle_insert": [vp, vp, vp, u64, vp],
            "oracle_find": [vp, vp, u64, vp, vp],
            "oracle_erase": [vp, vp, u64, vp],
            "oracle_mixed": [vp, vp, vp, vp, u64, vp, vp],
        }.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = ctypes.c_int
        L.oracle_get_stats.argtypes = [vp, ctypes.POINTER(_Stats)]
        L.oracle_dump.argtypes = [vp, vp, vp, u64]
        L.oracle_dump.restype = u64
        L.oracle_check.argtypes = [vp, ctypes.c_char_p, ctypes.c_int]
        L.oracle_check.restype = ctypes.c_int
        L.oracle_expand.argtypes = [vp, u32]
        L.oracle_contract.argtypes = [vp, u32]
        L.oracle_contract.restype = ctypes.c_int
        L.oracle_image.argtypes = [vp, vp, vp, u64]
        L.oracle_image.restype = u64
        L.oracle_bucket.argtypes = [vp, u64, vp]
        L.oracle_bucket.restype = u32
        L.oracle_pack.argtypes = [u32, u32]
        L.oracle_pack.restype = u64
        for n in ("oracle_unpack_key", "oracle_unpack_value"):
            getattr(L, n).argtypes = [u64]
            getattr(L, n).restype = u32
        for n in ("oracle_bithash1", "oracle_bithash2"):
            getattr(L, n).argtypes = [u32]
            getattr(L, n).restype = u32
        L.oracle_addr.argtypes = [u32, u32, u32]
        L.oracle_addr.restype = u32
        L.oracle_alt.argtypes = [u32, u32, u32, u32]
        L.oracle_alt.restype = u32
        L.oracle_ballot.argtypes = [vp]
        L.oracle_ballot.restype = u32
        L.oracle_first_set.argtypes = [u32]
        L.oracle_first_set.restype = ctypes.c_int
        L.oracle_prefix_rank.argtypes = [u32, u32]
        L.oracle_prefix_rank.restype = u32
        L.oracle_select_nth_one.argtypes = [u32, u32]
        L.oracle_select_nth_one.restype = ctypes.c_int
        L.oracle_crc32_bytes.argtypes = [vp, u64]
        L.oracle_crc32_bytes.restype = u32
        L.oracle_crc64_bytes.argtypes = [vp, u64]
        L.oracle_crc64_bytes.restype = u64
        for n in ("oracle_crc32", "oracle_crc64_lo"):
            getattr(L, n).argtypes = [u32]
            getattr(L, n).restype = u32
        L.oracle_set_hash.argtypes = [vp, u32]
        L.oracle_set_hash.restype = ctypes.c_int
        L.oracle_uniform_expected_collisions.argtypes = [u64, u64]
        L.oracle_uniform_expected_collisions.restype = ctypes.c_double
        L.oracle_observed_collisions.argtypes = [u32, vp, u64, u64]
        L.oracle_observed_collisions.restype = u64
        L.oracle_fmix32.argtypes = [u32]
        L.oracle_fmix32.restype = u32
        L.oracle_shard.argtypes = [u32, u32, u32]
        L.oracle_shard.restype = u32
        _lib = L
    return _lib


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleTable:
    """Sequential Hive table under the PHASED batch contract."""

    def __init__(self, capacity: int, max_capacity: int = 0, lf_grow: float = 0.9,
                 lf_shrink: float = 0.25, max_evictions: int = 16, resize_k: int = 1024,
                 stash_fraction: float = 0.02, hash: str = "bithash"):
        self._L = lib()
        self._h = self._L.oracle_create(capacity, max_capacity, lf_grow, lf_shrink,
                                        max_evictions, resize_k, stash_fraction)
        if self._L.oracle_set_hash(self._h, HASH_KINDS.get(hash, 99)) != 0:
            raise ValueError(hash)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._L.oracle_destroy(h)

    def insert(self, keys, vals) -> np.ndarray:
        k, v = _u32(keys), _u32(vals)
        st = np.zeros(len(k), np.uint8)
        self.rc = self._L.oracle_insert(self._h, _ptr(k), _ptr(v), len(k), _ptr(st))
        return st

    def find(self, keys):
        k = _u32(keys)
        vals = np.zeros(len(k), np.uint32)
        found = np.zeros(len(k), np.uint8)
        self._L.oracle_find(self._h, _ptr(k), len(k), _ptr(vals), _ptr(found))
        return vals, found

    def erase(self, keys) -> np.ndarray:
        k = _u32(keys)
        out = np.zeros(len(k), np.uint8)
        self._L.oracle_erase(self._h, _ptr(k), len(k), _ptr(out))
        return out

    def mixed(self, ops, keys, vals):
        o = np.ascontiguousarray(np.asarray(ops, dtype=np.uint8))
        k, v = _u32(keys), _u32(vals)
        vo = np.zeros(len(k), np.uint32)
        res = np.zeros(len(k), np.uint8)
        self.rc = self._L.oracle_mixed(self._h, _ptr(o), _ptr(k), _ptr(v), len(k), _ptr(vo), _ptr(res))
        return vo, res

    def stats(self) -> dict:
        s = _Stats()
        self._L.oracle_get_stats(self._h, ctypes.byref(s))
        return {n: getattr(s, n) for n, _ in _Stats._fields_}

    def dump(self):
        n = self._L.oracle_dump(self._h, None, None, 0)
        k = np.zeros(n, np.uint32)
        v = np.zeros(n, np.uint32)
        self._L.oracle_dump(self._h, _ptr(k), _ptr(v), n)
        return k, v

    def dump_dict(self) -> dict:
        k, v = self.dump()
        return dict(zip(k.tolist(), v.tolist()))

    def check(self) -> str:
        buf = ctypes.create_string_buffer(256)
        rc = self._L.oracle_check(self._h, buf, 256)
        return "" if rc == 0 else buf.value.decode()

    def expand(self, k: int):
        self._L.oracle_expand(self._h, k)

    def contract(self, k: int) -> bool:
        return bool(self._L.oracle_contract(self._h, k))

    def image(self):
        """(bucket array uint64[n_buckets * 32], live stash words uint64[k])."""
        nb = self.stats()["n_buckets"]
        slots = np.zeros(nb * 32, np.uint64)
        n = self._L.oracle_image(self._h, None, None, 0)
        stash = np.zeros(max(n, 1), np.uint64)
        self._L.oracle_image(self._h, _ptr(slots), _ptr(stash), n)
        return slots, stash[:n]

    def bucket(self, b: int):
        s = np.zeros(32, np.uint64)
        fm = self._L.oracle_bucket(self._h, b, _ptr(s))
        return s, fm


# --- primitives (for pins) ------------------------------------------------------
def pack(k, v): return lib().oracle_pack(k, v)
def unpack(p): return lib().oracle_unpack_key(p), lib().oracle_unpack_value(p)
HASH_KINDS = {"bithash": 0, "crc": 1}
HASH_FNS = {"bithash1": 0, "bithash2": 1, "crc32": 2, "crc64": 3}


def crc32_bytes(b: bytes) -> int:
    a = np.frombuffer(b, np.uint8).copy()
    return lib().oracle_crc32_bytes(_ptr(a), len(a))


def crc64_bytes(b: bytes) -> int:
    a = np.frombuffer(b, np.uint8).copy()
    return lib().oracle_crc64_bytes(_ptr(a), len(a))


def crc32(k): return lib().oracle_crc32(k)
def crc64_lo(k): return lib().oracle_crc64_lo(k)


def uniform_expected_collisions(n: int, m: int) -> float:
    """Theorem 1: E[Y] = n - m(1 - (1 - 1/m)^n)."""
    return lib().oracle_uniform_expected_collisions(n, m)


def observed_collisions(fn: str, keys, m: int) -> int:
    """Y = sum_b (L_b - 1)_+ with bin = hash(k) mod m."""
    k = _u32(keys)
    return lib().oracle_observed_collisions(HASH_FNS[fn], _ptr(k), len(k), m)


def csr(fn: str, keys, m: int) -> float:
    """Collision Speedup Ratio E[Y] / Y_observed."""
    return uniform_expected_collisions(len(keys), m) / observed_collisions(fn, keys, m)


def bithash1(k): return lib().oracle_bithash1(k)
def bithash2(k): return lib().oracle_bithash2(k)
def addr(h, mask, split): return lib().oracle_addr(h, mask, split)
def alt(key, cur, mask, split): return lib().oracle_alt(key, cur, mask, split)
def first_set(m): return lib().oracle_first_set(m)
def prefix_rank(m, lane): return lib().oracle_prefix_rank(m, lane)
def select_nth_one(m, r): return lib().oracle_select_nth_one(m, r)
def shard(key, seed, g): return lib().oracle_shard(key, seed, g)
def fmix32(h): return lib().oracle_fmix32(h)


def ballot(preds) -> int:
    p = np.ascontiguousarray(np.asarray(preds, dtype=np.uint8))
    assert p.shape == (32,)
    return lib().oracle_ballot(_ptr(p))


def shard_array(keys, seed: int, g: int) -> np.ndarray:
    L = lib()
    return np.array([L.oracle_shard(int(k), seed, g) for k in np.asarray(keys).tolist()], np.uint32)
