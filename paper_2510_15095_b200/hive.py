"""Thin ctypes binding over libhive.so (include/hive.h).

Argument marshalling only: torch tensors supply device memory and the current
CUDA stream; every step of the hot path runs in the library's sm_100a kernels.
There is no CPU fallback: without a built libhive.so or a CUDA device every
entry point raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libhive.so")

HIVE_KEYS_UNIQUE = 1
HIVE_HASH_CRC = 2
HIVE_SHARD_DEDUP = 4
HASH_PAIRS = {"bithash": 0, "crc": HIVE_HASH_CRC}      # (BitHash1, BitHash2) / (CRC-32, CRC-64)
HASH_FNS = {"bithash1": 0, "bithash2": 1, "crc32": 2, "crc64": 3}
OP_FIND, OP_INSERT, OP_ERASE = 0, 1, 2
INVALID_KEY = 0xFFFFFFFF

_STATUS = {0: "ok", 1: "invalid argument", 2: "out of memory", 3: "CUDA error", 4: "NCCL error",
           5: "stash full", 6: "handle busy", 7: "sharded exchange region full"}
SHARD_SEED = 0x5BD1E995                       # HIVE_SHARD_SEED


class HiveError(RuntimeError):
    pass


class HiveConfig(ctypes.Structure):
    _fields_ = [("capacity", ctypes.c_uint64), ("max_capacity", ctypes.c_uint64),
                ("lf_grow", ctypes.c_float), ("lf_shrink", ctypes.c_float),
                ("max_evictions", ctypes.c_uint32), ("resize_k", ctypes.c_uint32),
                ("stash_fraction", ctypes.c_float), ("flags", ctypes.c_uint32),
                ("nccl_comm", ctypes.c_void_p), ("shard_batch_max", ctypes.c_uint64),
                ("shard_slack", ctypes.c_float)]


class HiveStats(ctypes.Structure):
    _fields_ = [("n_buckets", ctypes.c_uint64), ("m", ctypes.c_uint32), ("split", ctypes.c_uint32)] + [
        (n, ctypes.c_uint64) for n in (
            "count", "stash_used", "stash_cap", "evictions", "max_depth", "stash_pushes", "leftovers",
            "grows", "shrinks", "merge_aborts", "failed", "in_b1", "mapped_bytes")] + [
        ("alg_bytes", ctypes.c_uint64 * 8)] + [
        ("step3", ctypes.c_uint64), ("xfail", ctypes.c_uint64), ("elect_overflow", ctypes.c_uint64),
        ("step_cycles", ctypes.c_uint64 * 4)]


# every exported symbol of include/hive.h, with its ctypes signature
_vp, _u32, _u64, _int = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
SIGNATURES = {
    "hive_config_default": (None, [ctypes.POINTER(HiveConfig)]),
    "hive_create": (_int, [ctypes.POINTER(HiveConfig), _vp, ctypes.POINTER(_vp)]),
    "hive_destroy": (_int, [_vp]),
    "hive_insert": (_int, [_vp, _vp, _vp, _u64, _vp, _vp]),
    "hive_find": (_int, [_vp, _vp, _u64, _vp, _vp, _vp]),
    "hive_erase": (_int, [_vp, _vp, _u64, _vp, _vp]),
    "hive_mixed": (_int, [_vp, _vp, _vp, _vp, _u64, _vp, _vp, _vp]),
    "hive_mixed_concurrent": (_int, [_vp, _vp, _vp, _vp, _u64, _vp, _vp, _vp]),
    "hive_clear": (_int, [_vp, _vp]),
    "hive_insert_host": (_int, [_vp, _vp, _vp, _u64, _vp, _vp]),
    "hive_find_host": (_int, [_vp, _vp, _u64, _vp, _vp, _vp]),
    "hive_size": (_int, [_vp, ctypes.POINTER(_u64)]),
    "hive_stats": (_int, [_vp, ctypes.POINTER(HiveStats)]),
    "hive_dump": (_int, [_vp, _vp, _vp, _u64, ctypes.POINTER(_u64), _vp]),
    "hive_profile": (_int, [_vp, _int]),
    "hive_load_image": (_int, [_vp, _vp, _u64, _vp, _u64, _vp]),
    "hive_profile_read": (_int, [_vp, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                                 ctypes.POINTER(_u64), _int, _int]),
    "hive_route": (_int, [_u32, _u32, _vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp]),
    "hive_route_keys": (_int, [_u32, _u32, _vp, _u64, _vp, _vp, _vp, _vp]),
    "hive_unroute": (_int, [_vp, _u64, _vp, _vp, _vp, _vp, _vp]),
    "hive_unpack_kv": (_int, [_vp, _u64, _vp, _vp, _vp]),
    "hive_hash": (_int, [_u32, _vp, _u64, _vp, _vp]),
    "hive_gather_ceiling": (_int, [_vp, _u64, _vp, _u64, _vp, _vp]),
    "hive_gather_ceiling_rw": (_int, [_vp, _u64, _vp, _u64, _vp, _u32, _vp]),
    "hive_route_p2p": (_int, [_u32, _u32, _u32, _vp, _vp, _vp, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hive_inbox_compact": (_int, [_u32, _u64, _vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp]),
    "hive_serve_inbox": (_int, [_vp, _u32, _u32, _u32, _u64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hive_unroute_pad": (_int, [_vp, _u64, _vp, _vp, _vp, _vp, ctypes.c_uint8, _vp, _vp]),
    "hive_return_p2p": (_int, [_u32, _u32, _u64, _vp, _u64, _vp, _vp, _vp, _vp, _vp]),
    "hive_p2p_signal": (_int, [_u32, _u32, _u32, _u64, _vp, _vp]),
    "hive_p2p_wait": (_int, [_u32, _u32, _u64, _vp, _u64, _vp]),
    "hive_dev_alloc": (_int, [_u64, ctypes.POINTER(_vp)]),
    "hive_dev_free": (_int, [_vp]),
    "hive_ipc_handle": (_int, [_vp, _vp]),
    "hive_ipc_open": (_int, [_vp, ctypes.POINTER(_vp)]),
    "hive_ipc_close": (_int, [_vp]),
    "hive_collisions": (_int, [_u32, _vp, _u64, _u64, ctypes.POINTER(_u64), _vp]),
    "hive_nccl_unique_id": (_int, [_vp]),
    "hive_nccl_comm_init": (_int, [_int, _int, _vp, ctypes.POINTER(_vp)]),
    "hive_nccl_comm_destroy": (_int, [_vp]),
    "hive_shard_info": (_int, [_vp, ctypes.POINTER(_int), ctypes.POINTER(_int), ctypes.POINTER(_u64)]),
    "hive_status_string": (ctypes.c_char_p, [_int]),
    "hive_last_error": (ctypes.c_char_p, []),
}

_lib = None


def lib():
    """Load libhive.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise HiveError(f"{LIB_PATH} is missing: run `python -m paper_2510_15095_b200.build` "
                            "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        detail = lib().hive_last_error().decode(errors="replace")
        raise HiveError(f"{what}: {_STATUS.get(rc, rc)} {detail}")


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev(t: torch.Tensor, nbytes_per: int) -> torch.Tensor:
    if not t.is_cuda:
        raise HiveError("expected a CUDA tensor")
    if t.element_size() != nbytes_per or not t.is_contiguous():
        raise HiveError(f"expected a contiguous {nbytes_per}-byte dtype tensor, got {t.dtype}")
    return t


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def u32(x, device="cuda") -> torch.Tensor:
    """uint32 tensor on `device` from numpy / list / tensor."""
    if isinstance(x, torch.Tensor):
        if x.element_size() == 4:
            return x.contiguous().view(torch.uint32).to(device)
        return x.to(torch.int64).to(torch.uint32).to(device)
    import numpy as np
    a = np.ascontiguousarray(np.asarray(x, dtype=np.uint32))
    return torch.from_numpy(a.view(np.int32)).view(torch.uint32).to(device)


def u8(x, device="cuda") -> torch.Tensor:
    import numpy as np
    if isinstance(x, torch.Tensor):
        return x.to(torch.uint8).to(device)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.uint8))).to(device)


class HiveTable:
    """One Hive table on the current CUDA device (a handle of include/hive.h)."""

    def __init__(self, capacity: int, max_capacity: int = 0, lf_grow: float = 0.9,
                 lf_shrink: float = 0.25, max_evictions: int = 16, resize_k: int = 1024,
                 stash_fraction: float = 0.02, keys_unique: bool = False, hash: str = "bithash",
                 stream=None, nccl_comm: int | None = None, shard_batch_max: int = 0,
                 shard_slack: float = 0.0625, shard_dedup: bool = False):
        """nccl_comm (an ncclComm_t from nccl_comm_init): create one shard of a
        hash-partitioned table; every op call is then collective over the comm
        (include/hive.h "Sharded tables")."""
        L = lib()
        if not torch.cuda.is_available():
            raise HiveError("no CUDA device: the Hive table runs only on the GPU")
        cfg = HiveConfig()
        L.hive_config_default(ctypes.byref(cfg))
        cfg.capacity, cfg.max_capacity = capacity, max_capacity
        cfg.lf_grow, cfg.lf_shrink = lf_grow, lf_shrink
        cfg.max_evictions, cfg.resize_k, cfg.stash_fraction = max_evictions, resize_k, stash_fraction
        cfg.flags = (HIVE_KEYS_UNIQUE if keys_unique else 0) | HASH_PAIRS[hash] | (HIVE_SHARD_DEDUP if shard_dedup else 0)
        cfg.nccl_comm = nccl_comm
        cfg.shard_batch_max, cfg.shard_slack = shard_batch_max, shard_slack
        self.cfg = cfg
        h = ctypes.c_void_p()
        _check(L.hive_create(ctypes.byref(cfg), ctypes.c_void_p(_stream(stream)), ctypes.byref(h)), "hive_create")
        self._h = h
        self._L = L

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            self._L.hive_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- device-resident batch ops --------------------------------------------------
    def insert(self, keys: torch.Tensor, vals: torch.Tensor, status: torch.Tensor | None = None,
               stream=None) -> torch.Tensor:
        keys, vals = _dev(keys, 4), _dev(vals, 4)
        n = keys.numel()
        if vals.numel() != n:
            raise HiveError("keys and vals differ in length")
        if status is None:
            status = torch.empty(n, dtype=torch.uint8, device=keys.device)
        _check(self._L.hive_insert(self._h, _p(keys), _p(vals), n, _p(status), _stream(stream)), "hive_insert")
        return status

    def find(self, keys: torch.Tensor, vals_out=None, found=None, stream=None):
        keys = _dev(keys, 4)
        n = keys.numel()
        if vals_out is None:
            vals_out = torch.empty(n, dtype=torch.uint32, device=keys.device)
        if found is None:
            found = torch.empty(n, dtype=torch.uint8, device=keys.device)
        _check(self._L.hive_find(self._h, _p(keys), n, _p(vals_out), _p(found), _stream(stream)), "hive_find")
        return vals_out, found

    def erase(self, keys: torch.Tensor, erased=None, stream=None) -> torch.Tensor:
        keys = _dev(keys, 4)
        n = keys.numel()
        if erased is None:
            erased = torch.empty(n, dtype=torch.uint8, device=keys.device)
        _check(self._L.hive_erase(self._h, _p(keys), n, _p(erased), _stream(stream)), "hive_erase")
        return erased

    def mixed(self, ops: torch.Tensor, keys: torch.Tensor, vals: torch.Tensor, vals_out=None,
              result=None, stream=None):
        ops, keys, vals = _dev(ops, 1), _dev(keys, 4), _dev(vals, 4)
        n = keys.numel()
        if vals_out is None:
            vals_out = torch.empty(n, dtype=torch.uint32, device=keys.device)
        if result is None:
            result = torch.empty(n, dtype=torch.uint8, device=keys.device)
        _check(self._L.hive_mixed(self._h, _p(ops), _p(keys), _p(vals), n, _p(vals_out), _p(result),
                                  _stream(stream)), "hive_mixed")
        return vals_out, result

    def mixed_concurrent(self, ops: torch.Tensor, keys: torch.Tensor, vals: torch.Tensor, vals_out=None,
                         result=None, stream=None):
        """hive_mixed_concurrent: the whole batch in one cooperative launch,
        linearizable per key (include/hive.h)."""
        ops, keys, vals = _dev(ops, 1), _dev(keys, 4), _dev(vals, 4)
        n = keys.numel()
        if vals_out is None:
            vals_out = torch.empty(n, dtype=torch.uint32, device=keys.device)
        if result is None:
            result = torch.empty(n, dtype=torch.uint8, device=keys.device)
        _check(self._L.hive_mixed_concurrent(self._h, _p(ops), _p(keys), _p(vals), n, _p(vals_out), _p(result),
                                             _stream(stream)), "hive_mixed_concurrent")
        return vals_out, result

    # ---- end-to-end variants: host tensors in, host tensors out -----------------------
    # (pinned host tensors; asynchronous on the current stream: results are valid
    # after torch.cuda.current_stream().synchronize())
    @staticmethod
    def _host(t: torch.Tensor, nbytes_per: int) -> torch.Tensor:
        if t.is_cuda or t.element_size() != nbytes_per or not t.is_contiguous():
            raise HiveError("expected a contiguous host tensor")
        return t

    def insert_host(self, keys_h, vals_h, status_h=None, stream=None):
        keys_h, vals_h = self._host(keys_h, 4), self._host(vals_h, 4)
        n = keys_h.numel()
        if status_h is None:
            status_h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        _check(self._L.hive_insert_host(self._h, _p(keys_h), _p(vals_h), n, _p(status_h), _stream(stream)),
               "hive_insert_host")
        return status_h

    def find_host(self, keys_h, vals_h=None, found_h=None, stream=None):
        keys_h = self._host(keys_h, 4)
        n = keys_h.numel()
        if vals_h is None:
            vals_h = torch.empty(n, dtype=torch.uint32, pin_memory=True)
        if found_h is None:
            found_h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        _check(self._L.hive_find_host(self._h, _p(keys_h), n, _p(vals_h), _p(found_h), _stream(stream)),
               "hive_find_host")
        return vals_h, found_h

    # ---- inspection -----------------------------------------------------------------
    def clear(self, stream=None):
        _check(self._L.hive_clear(self._h, _stream(stream)), "hive_clear")

    def size(self) -> int:
        n = ctypes.c_uint64()
        _check(self._L.hive_size(self._h, ctypes.byref(n)), "hive_size")
        return n.value

    def stats(self, allow_failed: bool = False) -> dict:
        s = HiveStats()
        rc = self._L.hive_stats(self._h, ctypes.byref(s))
        if not (allow_failed and rc in (5, 7)):
            _check(rc, "hive_stats")
        d = {n: getattr(s, n) for n, _ in HiveStats._fields_}
        d["alg_bytes"] = dict(zip(("find", "insert", "evict", "erase", "elect"), list(s.alg_bytes)[:5]))
        d["step_cycles"] = list(s.step_cycles)
        return d

    def dump(self):
        n = ctypes.c_uint64()
        _check(self._L.hive_dump(self._h, None, None, 0, ctypes.byref(n), _stream()), "hive_dump")
        k = torch.empty(max(n.value, 1), dtype=torch.uint32, device="cuda")
        v = torch.empty(max(n.value, 1), dtype=torch.uint32, device="cuda")
        _check(self._L.hive_dump(self._h, _p(k), _p(v), n.value, ctypes.byref(n), _stream()), "hive_dump")
        return k[:n.value], v[:n.value]

    def load_image(self, slots: torch.Tensor, stash: torch.Tensor | None = None, stream=None):
        """hive_load_image (test hook): slots = device uint64/int64 tensor of
        n_buckets * 32 packed words, stash = live stash words."""
        slots = _dev(slots, 8)
        n_st = 0 if stash is None else stash.numel()
        _check(self._L.hive_load_image(self._h, _p(slots), slots.numel() // 32,
                                       _p(_dev(stash, 8)) if n_st else None, n_st, _stream(stream)),
               "hive_load_image")

    def serve_inbox(self, kind: int, n_src: int, rank: int, region: int, inbox_kv: int, inbox_ops: int, cnt: int,
                    peer_res32, peer_res8, stream=None):
        """hive_serve_inbox: the owner's side of the peer-memory exchange with
        device-side counts (kind 0 find, 1 insert, 2 erase, 3 mixed)."""
        _check(self._L.hive_serve_inbox(self._h, kind, n_src, rank, region, ctypes.c_void_p(inbox_kv),
                                        ctypes.c_void_p(inbox_ops) if inbox_ops else None, ctypes.c_void_p(cnt),
                                        _ptrs(peer_res32), _ptrs(peer_res8), _stream(stream)), "hive_serve_inbox")

    def shard_info(self) -> tuple[int, int, int]:
        """(nranks, rank, padded exchange capacity per peer); (1, 0, 0) unsharded."""
        g, r, c = _int(), _int(), _u64()
        _check(self._L.hive_shard_info(self._h, ctypes.byref(g), ctypes.byref(r), ctypes.byref(c)),
               "hive_shard_info")
        return g.value, r.value, c.value

    def profile(self, enable: bool | int = True):
        """True / 1: per-kernel CUDA-event timing; 2: also the clock64 insertion
        step breakdown (stats()["step_cycles"])."""
        _check(self._L.hive_profile(self._h, int(enable)), "hive_profile")

    def profile_read(self, reset: bool = True) -> dict:
        m = 64
        names = (ctypes.c_char_p * m)()
        ms = (ctypes.c_double * m)()
        cnt = (ctypes.c_uint64 * m)()
        k = self._L.hive_profile_read(self._h, names, ms, cnt, m, 1 if reset else 0)
        return {names[i].decode(): (ms[i], cnt[i]) for i in range(min(k, m))}


# ---- routing for the hash-partitioned table ---------------------------
def route(keys: torch.Tensor, vals: torch.Tensor | None, ops: torch.Tensor | None, n_shards: int,
          seed: int, stream=None):
    """Stable partition of a batch by shard(k) = (fmix32(k ^ seed) * G) >> 32.
    Returns (send_kv int64[n] packed value<<32|key, send_ops uint8[n] | None,
    pos int32[n] (op i -> send position), counts int64[G])."""
    keys = _dev(keys, 4)
    n = keys.numel()
    dev = keys.device
    send_kv = torch.empty(n, dtype=torch.int64, device=dev)
    send_ops = torch.empty(n, dtype=torch.uint8, device=dev) if ops is not None else None
    pos = torch.empty(n, dtype=torch.int32, device=dev)
    counts = torch.empty(n_shards, dtype=torch.int64, device=dev)
    _check(lib().hive_route(n_shards, seed, _p(keys), _p(vals), _p(ops), n, _p(send_kv), _p(send_ops),
                            _p(pos), _p(counts), _stream(stream)), "hive_route")
    return send_kv, send_ops, pos, counts


def route_keys(keys: torch.Tensor, n_shards: int, seed: int, stream=None):
    """Keys-only stable partition: (send_keys uint32[n], pos int32[n], counts int64[G])."""
    keys = _dev(keys, 4)
    n = keys.numel()
    send = torch.empty(n, dtype=torch.uint32, device=keys.device)
    pos = torch.empty(n, dtype=torch.int32, device=keys.device)
    counts = torch.empty(n_shards, dtype=torch.int64, device=keys.device)
    _check(lib().hive_route_keys(n_shards, seed, _p(keys), n, _p(send), _p(pos), _p(counts), _stream(stream)),
           "hive_route_keys")
    return send, pos, counts


def unroute(pos: torch.Tensor, in8: torch.Tensor | None = None, in32: torch.Tensor | None = None,
            stream=None):
    n = pos.numel()
    out8 = torch.empty(n, dtype=torch.uint8, device=pos.device) if in8 is not None else None
    out32 = torch.empty(n, dtype=torch.uint32, device=pos.device) if in32 is not None else None
    _check(lib().hive_unroute(_p(pos), n, _p(in8), _p(out8), _p(in32), _p(out32), _stream(stream)),
           "hive_unroute")
    return out8, out32


def unpack_kv(kv: torch.Tensor, stream=None):
    n = kv.numel()
    k = torch.empty(n, dtype=torch.uint32, device=kv.device)
    v = torch.empty(n, dtype=torch.uint32, device=kv.device)
    _check(lib().hive_unpack_kv(_p(kv), n, _p(k), _p(v), _stream(stream)), "hive_unpack_kv")
    return k, v


def hash_keys(fn: str, keys: torch.Tensor, stream=None) -> torch.Tensor:
    """hive_hash: fn(keys) on the device (fn in HASH_FNS)."""
    n = keys.numel()
    out = torch.empty(n, dtype=torch.uint32, device=keys.device)
    _check(lib().hive_hash(HASH_FNS[fn], _p(keys), n, _p(out), _stream(stream)), "hive_hash")
    return out


def gather_ceiling(blocks: torch.Tensor, keys: torch.Tensor, out: torch.Tensor | None = None,
                   stream=None) -> torch.Tensor:
    """hive_gather_ceiling: random 256 B block reads at the lookup kernel's access
    pattern (SURVEY §8(d) calibration ceiling); blocks is a uint64 tensor of
    n_blocks * 32 words."""
    n = keys.numel()
    if out is None:
        out = torch.empty(n, dtype=torch.uint32, device=keys.device)
    _check(lib().hive_gather_ceiling(_p(blocks), blocks.numel() // 32, _p(keys), n, _p(out),
                                     _stream(stream)), "hive_gather_ceiling")
    return out


def gather_ceiling_rw(blocks: torch.Tensor, keys: torch.Tensor, mode: int, out: torch.Tensor | None = None,
                      stream=None) -> torch.Tensor:
    """hive_gather_ceiling_rw: the gather plus an 8 B store (mode 1) or a CAS
    (mode 2) into one slot per block -- an insert probe's read/write mix."""
    n = keys.numel()
    if out is None:
        out = torch.empty(n, dtype=torch.uint32, device=keys.device)
    _check(lib().hive_gather_ceiling_rw(_p(blocks), blocks.numel() // 32, _p(keys), n, _p(out), mode,
                                        _stream(stream)), "hive_gather_ceiling_rw")
    return out


def collisions(fn: str, keys: torch.Tensor, m: int, stream=None) -> int:
    """hive_collisions: Y = sum_b (L_b - 1)_+ over m bins (Theorem 1)."""
    y = _u64(0)
    _check(lib().hive_collisions(HASH_FNS[fn], _p(keys), keys.numel(), m, ctypes.byref(y),
                                 _stream(stream)), "hive_collisions")
    return int(y.value)


# ---- peer-memory exchange ----------------------------------------
def _ptrs(ptrs):
    """Host array of device pointers (ints) for the C ABI (None stays NULL)."""
    if ptrs is None:
        return None
    arr = (ctypes.c_void_p * len(ptrs))(*[ctypes.c_void_p(int(p)) if p else None for p in ptrs])
    return arr


def dev_alloc(nbytes: int) -> int:
    out = _vp()
    _check(lib().hive_dev_alloc(nbytes, ctypes.byref(out)), "hive_dev_alloc")
    return int(out.value)


def dev_free(ptr: int):
    _check(lib().hive_dev_free(ctypes.c_void_p(ptr)), "hive_dev_free")


def ipc_handle(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(lib().hive_ipc_handle(ctypes.c_void_p(ptr), buf), "hive_ipc_handle")
    return buf.raw


def ipc_open(handle: bytes) -> int:
    out = _vp()
    buf = ctypes.create_string_buffer(handle, 64)
    _check(lib().hive_ipc_open(buf, ctypes.byref(out)), "hive_ipc_open")
    return int(out.value)


def ipc_close(ptr: int):
    _check(lib().hive_ipc_close(ctypes.c_void_p(ptr)), "hive_ipc_close")


def route_p2p(n_shards, rank, seed, keys, vals, ops, region, peer_kv, peer_ops, peer_cnt, pos, counts,
              stream=None):
    n = keys.numel()
    _check(lib().hive_route_p2p(n_shards, rank, seed, _p(keys), _p(vals), _p(ops), n, region, _ptrs(peer_kv),
                                _ptrs(peer_ops), _ptrs(peer_cnt), _p(pos), _p(counts),
                                _stream(stream)), "hive_route_p2p")


def inbox_compact(n_src, region, inbox_kv: int, inbox_ops: int, cnt: int, n_total, keys, vals, ops,
                  stream=None):
    _check(lib().hive_inbox_compact(n_src, region, ctypes.c_void_p(inbox_kv),
                                    ctypes.c_void_p(inbox_ops) if inbox_ops else None, ctypes.c_void_p(cnt),
                                    n_total, _p(keys), _p(vals), _p(ops), _stream(stream)), "hive_inbox_compact")


def return_p2p(n_src, rank, region, cnt: int, n_total, res32, res8, peer_res32, peer_res8, stream=None):
    _check(lib().hive_return_p2p(n_src, rank, region, ctypes.c_void_p(cnt), n_total, _p(res32), _p(res8),
                                 _ptrs(peer_res32), _ptrs(peer_res8), _stream(stream)), "hive_return_p2p")


def unroute_raw(pos, n, in8: int, out8, in32: int, out32, stream=None):
    """hive_unroute with raw device pointers for the inputs (exchange buffers)."""
    _check(lib().hive_unroute(_p(pos), n, ctypes.c_void_p(in8) if in8 else None, _p(out8),
                              ctypes.c_void_p(in32) if in32 else None, _p(out32), _stream(stream)), "hive_unroute")


def unroute_pad_raw(pos, n, in8: int, out8, in32: int, out32, miss8: int, poison: int = 0, stream=None):
    """hive_unroute_pad with raw device pointers for the inputs."""
    _check(lib().hive_unroute_pad(_p(pos), n, ctypes.c_void_p(in8) if in8 else None, _p(out8),
                                  ctypes.c_void_p(in32) if in32 else None, _p(out32), miss8,
                                  ctypes.c_void_p(poison) if poison else None, _stream(stream)),
           "hive_unroute_pad")


def p2p_signal(n, rank, phase, epoch, peer_sig, stream=None):
    _check(lib().hive_p2p_signal(n, rank, phase, epoch, _ptrs(peer_sig), _stream(stream)), "hive_p2p_signal")


def p2p_wait(n, phase, epoch, sig: int, timeout_ns=60_000_000_000, stream=None):
    _check(lib().hive_p2p_wait(n, phase, epoch, ctypes.c_void_p(sig), timeout_ns, _stream(stream)), "hive_p2p_wait")


# ---- NCCL bootstrap for sharded tables ----------------------------------------------
def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().hive_nccl_unique_id(buf), "hive_nccl_unique_id")
    return buf.raw


def nccl_comm_init(nranks: int, rank: int, uid: bytes) -> int:
    out = _vp()
    buf = ctypes.create_string_buffer(uid, 128)
    _check(lib().hive_nccl_comm_init(nranks, rank, buf, ctypes.byref(out)), "hive_nccl_comm_init")
    return int(out.value)


def nccl_comm_destroy(comm: int):
    _check(lib().hive_nccl_comm_destroy(ctypes.c_void_p(comm)), "hive_nccl_comm_destroy")
