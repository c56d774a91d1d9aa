"""Erase throughput at cfg2 scale: 2^25 present keys (hits) and 2^25 absent
keys (misses) erased from a full 2^26-key table, per-kernel device times."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen
from paper_2510_15095_b200 import HiveTable, u32
n = 1 << 26
t = HiveTable(gen.CFG2_BUCKETS * 32, lf_grow=2.0, lf_shrink=0)
ids = np.arange(n, dtype=np.uint32)
k, v = u32(gen.keys_of(ids)), u32(gen.vals_of(ids))
miss = u32(gen.absent_keys(n // 2))
out = {}
for rep in range(3):
    t.clear(); t.insert(k, v); torch.cuda.synchronize()
    t.profile(True)
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record(); e = t.erase(k[: n // 2]); b.record(); m = t.erase(miss); c.record()
    torch.cuda.synchronize()
    p = t.profile_read(reset=True); t.profile(False)
    assert int(e.sum()) == n // 2 and int(m.sum()) == 0
    out = {"hit_gps": (n // 2) / (a.elapsed_time(b) * 1e-3) / 1e9,
           "miss_gps": (n // 2) / (b.elapsed_time(c) * 1e-3) / 1e9,
           "kern_ms": {kk: round(vv[0], 3) for kk, vv in p.items()}}
print(json.dumps(out))
