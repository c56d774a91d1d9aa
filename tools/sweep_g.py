"""Sweep lanes-per-op (G) for the probe kernels at cfg2 scale; prints ms per phase."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
from paper_2510_15095_b200 import HiveTable, u32
n = 1 << 26
ids = np.arange(n, dtype=np.uint32)
keys, vals = u32(gen.keys_of(ids)), u32(gen.vals_of(ids))
qids, hit = gen.mixed_queries(n // 2, n // 2, n, seed=202)
q = u32(gen.keys_of(qids))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
configs = [int(x) for x in (sys.argv[1:] or ["8", "4", "2", "1"])]
for uniq in (False, True):
    for g in configs:
        for k in ("HIVE_G_FIND", "HIVE_G_INSERT", "HIVE_G_ERASE", "HIVE_G_SLOW"):
            os.environ[k] = str(g)
        t = HiveTable(gen.CFG2_BUCKETS * 32, lf_grow=2.0, lf_shrink=0, keys_unique=uniq)
        t.profile(True)
        res = []
        for rep in range(3):
            t.clear()
            ev[0].record(); st = t.insert(keys, vals); ev[1].record()
            v, f = t.find(q); ev[2].record()
            e = t.erase(keys[: n // 2]); ev[3].record()
            torch.cuda.synchronize()
            res.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
        assert int((st != 0).sum()) == 0 and int(f.sum()) == n // 2 and int(e.sum()) == n // 2
        prof = t.profile_read()
        s = t.stats()
        r = np.array(res[1:]).mean(0)
        print(json.dumps({"G": g, "unique": uniq, "insert_ms": r[0], "find_ms": r[1], "erase_ms": r[2],
                          "kern": {k: round(v[0] / v[1], 3) for k, v in prof.items()},
                          "p_h1": s["in_b1"] / (s["count"] - s["stash_used"] + 1e-9),
                          "evictions": s["evictions"], "leftovers": s["leftovers"]}), flush=True)
        del t
