"""k_dedup_elect time vs batch size (election table 16n bytes: L2-resident up to ~2^22)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen
from paper_2510_15095_b200 import HiveTable, u32
for lg in (18, 20, 21, 22, 23, 24, 26):
    n = 1 << lg
    t = HiveTable(-(-n * 100 // (95 * 32)) * 32, lf_grow=2.0, lf_shrink=0)
    k = u32(gen.present_keys(n)); v = u32(gen.vals_of(np.arange(n)))
    for _ in range(2):
        t.clear(); t.insert(k, v)
    t.profile(True)
    for _ in range(3):
        t.clear(); t.insert(k, v)
    torch.cuda.synchronize()
    p = t.profile_read()
    e = p["k_dedup_elect"]
    f = p["k_insert_fast"]
    print(json.dumps({"log2n": lg, "elect_ms": e[0] / e[1], "elect_Gops": n / (e[0] / e[1] * 1e-3) / 1e9,
                      "fast_ms": f[0] / f[1], "fast_Gops": n / (f[0] / f[1] * 1e-3) / 1e9}), flush=True)
    del t
