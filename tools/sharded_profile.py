"""Stage timings of the sharded path at world size 1 (NCCL loopback)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29555")
import numpy as np, torch, torch.distributed as dist
import gen
from paper_2510_15095_b200 import u32
from paper_2510_15095_b200.sharded import ShardedHive
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = 1 << 26
ids = np.arange(n, dtype=np.uint32)
keys, vals = u32(gen.keys_of(ids)), u32(gen.vals_of(ids))
qids, _ = gen.mixed_queries(n // 2, n // 2, n, seed=202)
q = u32(gen.keys_of(qids))
sh = ShardedHive(gen.CFG2_BUCKETS * 32, lf_grow=2.0, lf_shrink=0)
T = {}
def tm(name, f):
    torch.cuda.synchronize(); a = time.perf_counter(); r = f(); torch.cuda.synchronize()
    T[name] = T.get(name, 0) + (time.perf_counter() - a) * 1e3
    return r
for rep in range(3):
    if rep == 1: T.clear()
    sh.table.clear()
    send_kv, _, pos, counts = tm("ins.route", lambda: sh.ops.route(keys, vals, None, 1, sh.seed))
    sc, rc = tm("ins.counts", lambda: sh._counts(counts))
    recv = tm("ins.a2a_fwd", lambda: sh._a2a(send_kv, rc, sc))
    k, v = tm("ins.unpack", lambda: sh.ops.unpack(recv))
    st = tm("ins.local", lambda: sh.table.insert(k, v))
    back = tm("ins.a2a_back", lambda: sh._a2a_u8(st, sc, rc))
    tm("ins.unroute", lambda: sh.ops.unroute(pos, in8=back))
    send_kv, _, pos, counts = tm("find.route", lambda: sh.ops.route(q, None, None, 1, sh.seed))
    sc, rc = tm("find.counts", lambda: sh._counts(counts))
    recv = tm("find.a2a_fwd", lambda: sh._a2a(send_kv, rc, sc))
    k, _ = tm("find.unpack", lambda: sh.ops.unpack(recv))
    vv, ff = tm("find.local", lambda: sh.table.find(k))
    bv = tm("find.a2a_back", lambda: (sh._a2a_u32(vv, sc, rc), sh._a2a_u8(ff, sc, rc)))
    tm("find.unroute", lambda: sh.ops.unroute(pos, in8=bv[1], in32=bv[0]))
print({k: round(v / 2, 3) for k, v in T.items()})
print("total ms", round(sum(T.values()) / 2, 3))
dist.destroy_process_group()
