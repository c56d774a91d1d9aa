"""Hash-partitioned table, N > 1 path, on CPU: world size 2 over gloo.

`ShardedHive` (the product's exchange logic: route -> all-to-all of counts and
records -> local phases -> inverse all-to-all -> unpermute) runs unchanged;
only the device primitives are replaced by an oracle-backed stand-in (routing
by the oracle's shard function, a stable sort, and an OracleTable per rank).
Expected results are computed independently in the parent: shard s processes
the rank-major concatenation of the ops routed to it."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SEED = 0x5BD1E995
WORLD = 2


class OracleTableAdapter:
    def __init__(self, capacity, **cfg):
        import oracle
        self.t = oracle.OracleTable(capacity, **cfg)

    @staticmethod
    def _np(x):
        return x.numpy().view(np.uint32) if x.dtype in (torch.uint32, torch.int32) else x.numpy()

    def insert(self, k, v):
        return torch.from_numpy(self.t.insert(self._np(k), self._np(v)))

    def find(self, k):
        v, f = self.t.find(self._np(k))
        return torch.from_numpy(v.view(np.int32)).view(torch.uint32), torch.from_numpy(f)

    def erase(self, k):
        return torch.from_numpy(self.t.erase(self._np(k)))

    def mixed(self, o, k, v):
        vo, r = self.t.mixed(o.numpy(), self._np(k), self._np(v))
        return torch.from_numpy(vo.view(np.int32)).view(torch.uint32), torch.from_numpy(r)


class OracleOps:
    """CPU stand-in for hive_route / hive_unroute / hive_unpack_kv."""

    def __init__(self, capacity, **cfg):
        self.table = OracleTableAdapter(capacity, **cfg)

    @staticmethod
    def route(keys, vals, ops, n_shards, seed):
        import oracle
        k = keys.numpy().view(np.uint32)
        sh = oracle.shard_array(k, seed, n_shards)
        order = np.argsort(sh, kind="stable")
        v = vals.numpy().view(np.uint32) if vals is not None else np.zeros_like(k)
        kv = (v[order].astype(np.uint64) << np.uint64(32)) | k[order].astype(np.uint64)
        pos = np.empty(len(k), np.int32)
        pos[order] = np.arange(len(k), dtype=np.int32)
        send_ops = torch.from_numpy(ops.numpy()[order].copy()) if ops is not None else None
        counts = torch.from_numpy(np.bincount(sh, minlength=n_shards).astype(np.int64))
        return torch.from_numpy(kv.view(np.int64)), send_ops, torch.from_numpy(pos), counts

    @staticmethod
    def route_keys(keys, n_shards, seed):
        import oracle
        k = keys.numpy().view(np.uint32)
        sh = oracle.shard_array(k, seed, n_shards)
        order = np.argsort(sh, kind="stable")
        pos = np.empty(len(k), np.int32)
        pos[order] = np.arange(len(k), dtype=np.int32)
        counts = torch.from_numpy(np.bincount(sh, minlength=n_shards).astype(np.int64))
        return _t32(k[order]), torch.from_numpy(pos), counts

    @staticmethod
    def unroute(pos, in8=None, in32=None):
        p = pos.numpy()
        o8 = torch.from_numpy(in8.numpy()[p].copy()) if in8 is not None else None
        o32 = None
        if in32 is not None:
            o32 = torch.from_numpy(in32.numpy().view(np.int32)[p].copy()).view(torch.uint32)
        return o8, o32

    @staticmethod
    def unpack(kv):
        w = kv.numpy().view(np.uint64)
        k = (w & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        v = (w >> np.uint64(32)).astype(np.uint32)
        return (torch.from_numpy(k.view(np.int32)).view(torch.uint32),
                torch.from_numpy(v.view(np.int32)).view(torch.uint32))


def _batches(rank):
    rng = np.random.default_rng(100 + rank)
    out = []
    for b in range(4):
        n = int(rng.integers(200, 3000))
        keys = rng.integers(0, 4000, n, dtype=np.uint64).astype(np.uint32)   # cross-rank duplicates
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        ops = rng.integers(0, 3, n).astype(np.uint8)
        out.append(("insert" if b == 0 else "mixed", ops, keys, vals))
    out.append(("find", None, rng.integers(0, 5000, 2000, dtype=np.uint64).astype(np.uint32), None))
    out.append(("erase", None, rng.integers(0, 5000, 1000, dtype=np.uint64).astype(np.uint32), None))
    return out


def _t32(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).view(torch.uint32)


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2510_15095_b200.sharded import ShardedHive
    sh = ShardedHive(ops=OracleOps(64 * 32, resize_k=16), seed=SEED)
    res = []
    for kind, ops, keys, vals in _batches(rank):
        if kind == "insert":
            r = sh.insert(_t32(keys), _t32(vals))
            res.append((r.numpy().copy(),))
        elif kind == "mixed":
            vo, r = sh.mixed(torch.from_numpy(ops), _t32(keys), _t32(vals))
            res.append((r.numpy().copy(), vo.numpy().view(np.uint32).copy()))
        elif kind == "find":
            v, f = sh.find(_t32(keys))
            res.append((f.numpy().copy(), v.numpy().view(np.uint32).copy()))
        else:
            r = sh.erase(_t32(keys))
            res.append((r.numpy().copy(),))
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def _expected():
    """Independent expectation: per-shard oracles over rank-major sequences."""
    import oracle
    shards = [oracle.OracleTable(64 * 32, resize_k=16) for _ in range(WORLD)]
    per_rank = [_batches(r) for r in range(WORLD)]
    exp = [[] for _ in range(WORLD)]
    for b in range(len(per_rank[0])):
        kind = per_rank[0][b][0]
        outs = [dict() for _ in range(WORLD)]
        for s in range(WORLD):
            cat_ops, cat_keys, cat_vals, owners = [], [], [], []
            for r in range(WORLD):
                _, ops, keys, vals = per_rank[r][b]
                sh = oracle.shard_array(keys, SEED, WORLD)
                idx = np.flatnonzero(sh == s)
                cat_keys.append(keys[idx])
                cat_vals.append(vals[idx] if vals is not None else np.zeros(len(idx), np.uint32))
                cat_ops.append(ops[idx] if ops is not None else np.zeros(len(idx), np.uint8))
                owners += [(r, int(i)) for i in idx]
            k, v, o = np.concatenate(cat_keys), np.concatenate(cat_vals), np.concatenate(cat_ops)
            if kind == "insert":
                res = (shards[s].insert(k, v),)
            elif kind == "mixed":
                vo, rr = shards[s].mixed(o, k, v)
                res = (rr, vo)
            elif kind == "find":
                vv, ff = shards[s].find(k)
                res = (ff, vv)
            else:
                res = (shards[s].erase(k),)
            for j, (r, i) in enumerate(owners):
                outs[r][i] = tuple(x[j] for x in res)
        for r in range(WORLD):
            n = len(per_rank[r][b][2])
            exp[r].append(tuple(np.array([outs[r][i][c] for i in range(n)]) for c in range(len(outs[r][0]))))
    return exp


@pytest.mark.timeout(300)
def test_sharded_exchange_world2_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    exp = _expected()
    for r in range(WORLD):
        assert len(got[r]) == len(exp[r])
        for b, (g, e) in enumerate(zip(got[r], exp[r])):
            for gc, ec in zip(g, e):
                assert (np.asarray(gc).astype(np.int64) == np.asarray(ec).astype(np.int64)).all(), (r, b)
