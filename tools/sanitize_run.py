"""Small mixed workload for compute-sanitizer (insert/find/erase/mixed with
growth, shrink, duplicates, stash)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen
from paper_2510_15095_b200 import HiveTable, u8, u32
t = HiveTable(64 * 32, resize_k=8)
rng = np.random.default_rng(3)
for b in range(6):
    n = 4000
    ops = gen.bernoulli_ops(n, 0.5, 0.2, seed=b)
    keys = rng.integers(0, 6000, n, dtype=np.uint64).astype(np.uint32)
    t.mixed(u8(ops), u32(keys), u32(keys ^ 7))
k = u32(gen.present_keys(5000))
t.insert(k, k); t.find(k); t.erase(k[:4000])
u = HiveTable(16 * 32, lf_grow=2.0, lf_shrink=0)        # overfull: Steps 3-4
kk = u32(gen.present_keys(16 * 32 + 200))
u.insert(kk, kk); u.find(kk); u.erase(kk[:100])
torch.cuda.synchronize()
print("ok", t.size(), u.size())
