"""Hash-partitioned Hive table: one shard per GPU.

Each rank owns an independent Hive table (its own resize, stash and
counters).  A batch is routed by shard(k) = (fmix32(k ^ seed) * G) >> 32
with the stable partition kernel (hive_route), exchanged with an all-to-all
(NCCL over NVLink/NVSwitch on GPUs; any torch.distributed backend works),
processed by the owner shard, and the per-op results come back through the
inverse all-to-all and the unpermute kernel (hive_unroute).

Ordering: the receive buffer concatenates source ranks in rank order and the
route is stable, so a shard sees the union batch in (rank, local index) order;
in-batch duplicates across ranks therefore resolve to the op with the largest
(rank, index) — the "last write" of the rank-major global order.

`ops` is the device-side primitive set.  `CudaOps` (the product) calls the
C ABI; tests on CPU (gloo) substitute an equivalent test implementation to
exercise the exchange logic without a GPU.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import hive

SHARD_SEED = 0x5BD1E995


class CudaOps:
    """Routing primitives and a local table, all on the GPU via libhive.so."""

    def __init__(self, capacity: int, **cfg):
        self.table = hive.HiveTable(capacity, **cfg)

    @staticmethod
    def route(keys, vals, ops, n_shards, seed):
        return hive.route(keys, vals, ops, n_shards, seed)

    @staticmethod
    def route_keys(keys, n_shards, seed):
        return hive.route_keys(keys, n_shards, seed)

    @staticmethod
    def unroute(pos, in8=None, in32=None):
        return hive.unroute(pos, in8=in8, in32=in32)

    @staticmethod
    def unpack(kv):
        return hive.unpack_kv(kv)


class ShardedHive:
    def __init__(self, capacity_per_shard: int = 0, group=None, seed: int = SHARD_SEED,
                 ops=None, **cfg):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.seed = seed
        self.ops = ops if ops is not None else CudaOps(capacity_per_shard, **cfg)
        self.table = self.ops.table

    # ---- exchange ---------------------------------------------------------------
    def _counts(self, send_counts: torch.Tensor):
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        both = torch.stack([send_counts, recv_counts]).cpu()   # one small D2H per batch
        return both[0].tolist(), both[1].tolist()

    def _a2a(self, x: torch.Tensor, out_splits, in_splits) -> torch.Tensor:
        out = torch.empty(sum(out_splits), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(out, x, out_splits, in_splits, group=self.group)
        return out

    def _a2a_u8(self, x, out_splits, in_splits):
        return self._a2a(x, out_splits, in_splits)

    def _a2a_u32(self, x, out_splits, in_splits):
        # int32 view: every backend supports it
        y = self._a2a(x.view(torch.int32), out_splits, in_splits)
        return y.view(torch.uint32)

    def _forward(self, keys, vals, ops_codes):
        send_kv, send_ops, pos, counts = self.ops.route(keys, vals, ops_codes, self.world, self.seed)
        sc, rc = self._counts(counts)
        recv_kv = self._a2a(send_kv, rc, sc)
        recv_ops = self._a2a_u8(send_ops, rc, sc) if send_ops is not None else None
        k, v = self.ops.unpack(recv_kv)
        return k, v, recv_ops, pos, sc, rc

    # ---- collective batch ops (every rank calls with its own local batch) -----------
    def insert(self, keys, vals):
        k, v, _, pos, sc, rc = self._forward(keys, vals, None)
        st = self.table.insert(k, v)
        back = self._a2a_u8(st, sc, rc)
        out8, _ = self.ops.unroute(pos, in8=back)
        return out8

    def _forward_keys(self, keys):
        send, pos, counts = self.ops.route_keys(keys, self.world, self.seed)
        sc, rc = self._counts(counts)
        return self._a2a_u32(send, rc, sc), pos, sc, rc

    def find(self, keys):
        k, pos, sc, rc = self._forward_keys(keys)
        vals, found = self.table.find(k)
        bv = self._a2a_u32(vals, sc, rc)
        bf = self._a2a_u8(found, sc, rc)
        f, v = self.ops.unroute(pos, in8=bf, in32=bv)
        return v, f

    def erase(self, keys):
        k, pos, sc, rc = self._forward_keys(keys)
        er = self.table.erase(k)
        back = self._a2a_u8(er, sc, rc)
        out8, _ = self.ops.unroute(pos, in8=back)
        return out8

    def mixed(self, op_codes, keys, vals):
        k, v, o, pos, sc, rc = self._forward(keys, vals, op_codes)
        vals_out, result = self.table.mixed(o, k, v)
        bv = self._a2a_u32(vals_out, sc, rc)
        br = self._a2a_u8(result, sc, rc)
        r, vo = self.ops.unroute(pos, in8=br, in32=bv)
        return vo, r
