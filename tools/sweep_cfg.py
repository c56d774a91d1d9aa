"""Time insert / find / erase at cfg2 scale for several env configurations
(HIVE_G_*, HIVE_MINB).  Usage: sweep_cfg.py 'G_INSERT=4,MINB=1' 'G_INSERT=4,MINB=4' ..."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen
from paper_2510_15095_b200 import HiveTable, u32
n = 1 << 26
ids = np.arange(n, dtype=np.uint32)
keys, vals = u32(gen.keys_of(ids)), u32(gen.vals_of(ids))
qids, hit = gen.mixed_queries(n // 2, n // 2, n, seed=202)
q = u32(gen.keys_of(qids))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for spec in sys.argv[1:]:
    for item in spec.split(","):
        k, v = item.split("=")
        os.environ["HIVE_" + k] = v
    uniq = os.environ.get("HIVE_UNIQ") == "1"
    t = HiveTable(gen.CFG2_BUCKETS * 32, lf_grow=2.0, lf_shrink=0, keys_unique=uniq)
    t.profile(True)
    res = []
    for rep in range(4):
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
    print(json.dumps({"cfg": spec, "insert_ms": round(r[0], 3), "find_ms": round(r[1], 3), "erase_ms": round(r[2], 3),
                      "kern": {k: round(v[0] / v[1], 3) for k, v in prof.items()},
                      "evictions": s["evictions"], "leftovers": s["leftovers"]}), flush=True)
    del t
