"""Hash-partitioned Hive table: one shard per GPU.

Each rank owns an independent Hive table (its own resize, stash and
counters).  Key k belongs to rank shard(k) = (fmix32(k ^ seed) * G) >> 32.

`ShardedHive` is the C-ABI sharded handle (NCCL inside the library, padded
all-to-all, no host synchronisation with growth off).  `P2PShardedHive`
 moves records and results with the kernels' own stores
over NVLink peer mappings instead of NCCL.

Ordering: a shard sees the union batch in (rank, local index) order; in-batch
duplicates across ranks therefore resolve to the op with the largest
(rank, index) — the "last write" of the rank-major global order.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

from . import hive

SHARD_SEED = hive.SHARD_SEED


class ShardedHive:
    """One rank's shard of a hash-partitioned Hive table behind the C ABI
    (include/hive.h "Sharded tables"): argument marshalling only.  The NCCL
    comm is made by the library (hive_nccl_unique_id on rank 0, broadcast over
    the torch.distributed group, hive_nccl_comm_init on every rank); routing,
    the padded ncclAlltoAll exchange, the owner's PHASED batch and the inverse
    exchange all run inside the library on the current stream.  Every op is
    collective: each rank passes its own local batch (<= batch_max ops)."""

    def __init__(self, capacity_per_shard: int, batch_max: int, group=None, slack: float = 0.0625, **cfg):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        obj = [hive.nccl_unique_id() if self.rank == 0 else None]
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(obj, src=src, group=group)
        self.comm = hive.nccl_comm_init(self.world, self.rank, obj[0])
        self.table = hive.HiveTable(capacity_per_shard, nccl_comm=self.comm, shard_batch_max=batch_max,
                                    shard_slack=slack, **cfg)
        self.seed = SHARD_SEED

    def close(self):
        if getattr(self, "table", None) is not None:
            self.table.close()
            self.table = None
            hive.nccl_comm_destroy(self.comm)

    def insert(self, keys, vals, status=None):
        return self.table.insert(keys, vals, status)

    def find(self, keys, vals_out=None, found=None):
        return self.table.find(keys, vals_out, found)

    def erase(self, keys, erased=None):
        return self.table.erase(keys, erased)

    def mixed(self, op_codes, keys, vals, vals_out=None, result=None):
        return self.table.mixed(op_codes, keys, vals, vals_out, result)

    def insert_host(self, keys_h, vals_h, status_h=None):
        return self.table.insert_host(keys_h, vals_h, status_h)

    def find_host(self, keys_h, vals_h=None, found_h=None):
        return self.table.find_host(keys_h, vals_h, found_h)


# ---- NEXT-1: exchange over NVLink peer memory (no NCCL on the data path) -------------
class _DevView:
    """Zero-copy torch view of a raw device allocation (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _view(ptr: int, n: int, dtype: torch.dtype) -> torch.Tensor:
    ts = {torch.uint8: "|u1", torch.int32: "<i4", torch.int64: "<i8"}[dtype]
    return torch.as_tensor(_DevView(ptr, n, ts), device="cuda")


class PeerBuffers:
    """One rank's exchange buffers (plain cudaMalloc: IPC-exportable), laid out
    in `region`-sized per-rank regions (include/hive.h, NEXT-1)."""

    FIELDS = (("kv", 8), ("ops", 1), ("cnt", 0), ("res32", 4), ("res8", 1), ("sig", 0))
    SIG_WORDS = 17                           # [2 phases][8 sources] epochs + timeout marker

    def __init__(self, world: int, region: int):
        self.world, self.region = world, region
        self.ptr = {}
        for name, width in self.FIELDS:
            nbytes = {"cnt": world * 8, "sig": self.SIG_WORDS * 8}.get(name, world * region * width)
            self.ptr[name] = hive.dev_alloc(nbytes)
        _view(self.ptr["sig"], self.SIG_WORDS, torch.int64).zero_()
        _view(self.ptr["cnt"], world, torch.int64).zero_()
        torch.cuda.synchronize()
        self.owned = True

    @classmethod
    def mapped(cls, world: int, region: int, ptrs: dict):
        b = cls.__new__(cls)
        b.world, b.region, b.ptr, b.owned = world, region, dict(ptrs), False
        return b

    def handles(self) -> dict:
        return {k: hive.ipc_handle(v) for k, v in self.ptr.items()}

    def close(self):
        for v in self.ptr.values():
            (hive.dev_free if self.owned else hive.ipc_close)(v)
        self.ptr = {}


class P2PShardedHive:
    """Hash-partitioned table whose exchange is done by the kernels themselves:
    hive_route_p2p stores each op record straight into its owner's inbox over
    NVLink; hive_serve_inbox compacts the inbox by its DEVICE-side counts, runs
    one PHASED batch and stores each result straight back into its source's
    result region; the source's hive_unroute_pad restores its op order.  The
    phases are ordered by device-side signals (hive_p2p_signal / hive_p2p_wait:
    release stores into the peers' signal words, acquire spins): with growth
    off a call has no host synchronisation at all.  A peer that never signals
    sets the timeout marker, which the unroute kernel turns into result 6 for
    every op of that call (check() raises and resets it).  Same semantics as
    ShardedHive: a shard sees the union batch in (rank, index) order.

    `region` = records per (source, owner) region; padded_region(batch_max,
    world) sizes it like the NCCL path (batch / world * (1 + slack) + 1024), so
    the buffers cost ~1/world of one region per batch op; an op past its region
    is not sent (result 4, find found 2).

    `virtual_group` builds `world` ranks inside ONE process on one GPU (the
    peers' buffers are then plain local pointers): the tests drive the phases
    of all virtual ranks in lockstep to check the multi-rank logic."""

    KIND = {"find": 0, "insert": 1, "erase": 2, "mixed": 3}        # hive_serve_inbox kinds

    @staticmethod
    def padded_region(batch_max: int, world: int, slack: float = 0.0625) -> int:
        """Records per (source, owner) region: the NCCL handle's per-peer capacity."""
        if world <= 1:
            return int(batch_max)
        return int(min(batch_max, math.ceil(batch_max * (1 + slack) / world) + 1024))

    def __init__(self, capacity_per_shard: int, region: int, group=None, seed: int = SHARD_SEED,
                 _virtual=None, **cfg):
        self.seed, self.region, self.group = seed, region, group
        self._virtual = _virtual is not None
        if _virtual is None:
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
            self.own = PeerBuffers(self.world, region)
            hs = [None] * self.world
            dist.all_gather_object(hs, self.own.handles(), group=group)
            self.peers = [self.own if r == self.rank else
                          PeerBuffers.mapped(self.world, region, {k: hive.ipc_open(h) for k, h in hs[r].items()})
                          for r in range(self.world)]
        else:
            self.rank, self.world, self.peers = _virtual
            self.own = self.peers[self.rank]
        if self.world > 8:
            raise hive.HiveError("peer-memory exchange supports at most 8 shards (one node)")
        self.table = hive.HiveTable(capacity_per_shard, **cfg)
        self._state = None
        self._epoch = 0
        self.timeout_ns = 60_000_000_000          # a phase wait gives up after this (then results are 6)
        if _virtual is None:
            dist.barrier(group=group)       # every rank's signal words are zeroed

    @classmethod
    def virtual_group(cls, world: int, capacity_per_shard: int, region: int, **cfg):
        bufs = [PeerBuffers(world, region) for _ in range(world)]
        return [cls(capacity_per_shard, region, _virtual=(r, world, bufs), **cfg) for r in range(world)]

    def close(self):
        if self._virtual:                 # every virtual rank frees only its own buffers
            self.own.close()
        else:
            for p in self.peers:
                p.close()                 # peers: IPC unmap; own: free
        self.table.close()

    def _col(self, name):
        return [p.ptr[name] for p in self.peers]

    # ---- the three phases (every rank runs each phase before any runs the next) ----
    def route_phase(self, kind: str, keys, vals=None, ops=None):
        n = keys.numel()
        if vals is None:
            vals = torch.zeros(n, dtype=torch.uint32, device=keys.device)
        pos = torch.empty(n, dtype=torch.uint32, device=keys.device)
        counts = torch.empty(self.world, dtype=torch.int64, device=keys.device)
        self._epoch += 1
        hive.route_p2p(self.world, self.rank, self.seed, keys, vals, ops, self.region, self._col("kv"),
                       self._col("ops") if ops is not None else None, self._col("cnt"), pos, counts)
        hive.p2p_signal(self.world, self.rank, 0, self._epoch, self._col("sig"))
        self._state = (kind, n, pos)

    def check(self):
        """Raise (and reset the marker) if a peer missed a phase signal; the
        calls themselves never wait on the host for it (results of such a call
        are all 6)."""
        sig = _view(self.own.ptr["sig"], PeerBuffers.SIG_WORDS, torch.int64)
        if int(sig[-1].item()):
            sig[-1].zero_()                     # reset the marker: the handle stays usable
            self._state = None
            raise hive.HiveError("peer exchange: a peer did not signal within the timeout")

    def serve_phase(self):
        kind = self._state[0]
        hive.p2p_wait(self.world, 0, self._epoch, self.own.ptr["sig"], self.timeout_ns)   # all records are in
        vals32 = kind in ("find", "mixed")
        self.table.serve_inbox(self.KIND[kind], self.world, self.rank, self.region, self.own.ptr["kv"],
                               self.own.ptr["ops"] if kind == "mixed" else 0, self.own.ptr["cnt"],
                               self._col("res32") if vals32 else None, self._col("res8"))
        hive.p2p_signal(self.world, self.rank, 1, self._epoch, self._col("sig"))

    def finish_phase(self):
        kind, n, pos = self._state
        self._state = None
        dev = pos.device
        hive.p2p_wait(self.world, 1, self._epoch, self.own.ptr["sig"], self.timeout_ns)   # all results are back
        out8 = torch.empty(n, dtype=torch.uint8, device=dev)
        out32 = torch.empty(n, dtype=torch.uint32, device=dev) if kind in ("find", "mixed") else None
        if n:
            # the timeout marker poisons the results instead of a host check
            hive.unroute_pad_raw(pos, n, self.own.ptr["res8"], out8,
                                 self.own.ptr["res32"] if out32 is not None else 0, out32,
                                 2 if kind == "find" else 4, self.own.ptr["sig"] + 8 * (PeerBuffers.SIG_WORDS - 1))
        return out8, out32

    def _call(self, kind, keys, vals=None, ops=None):
        # no host barrier and no host synchronisation: the phases are ordered
        # by the device-side signals, the owner works from device-side counts
        self.route_phase(kind, keys, vals, ops)
        self.serve_phase()
        return self.finish_phase()

    # ---- collective batch ops (every rank calls with its own local batch) -----------
    def insert(self, keys, vals):
        return self._call("insert", keys, vals)[0]

    def erase(self, keys):
        return self._call("erase", keys)[0]

    def find(self, keys):
        f, v = self._call("find", keys)
        return v, f

    def mixed(self, op_codes, keys, vals):
        r, vo = self._call("mixed", keys, vals, op_codes)
        return vo, r
