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
# NEXT-4 monolithic kernel (cooperative launch) and the NEXT-2 clock64 variants
for b in range(3):
    n = 3000
    keys = rng.integers(0, 4000, n, dtype=np.uint64).astype(np.uint32)
    t.mixed_concurrent(u8(gen.bernoulli_ops(n, 0.4, 0.2, seed=50 + b)), u32(keys), u32(keys ^ 9))
t.profile(2)
t.insert(u32(gen.present_keys(6000)), u32(gen.present_keys(6000)))
t.profile(False)
u = HiveTable(16 * 32, lf_grow=2.0, lf_shrink=0)        # overfull: Steps 3-4
kk = u32(gen.present_keys(16 * 32 + 200))
u.insert(kk, kk); u.find(kk); u.erase(kk[:100])
# peer-memory exchange (NEXT-1) with 3 virtual ranks, and the calibration gather
from paper_2510_15095_b200 import hive
from paper_2510_15095_b200.sharded import P2PShardedHive
ranks = P2PShardedHive.virtual_group(3, 32 * 32, 3000, resize_k=8)
for kind in ("mixed", "find"):
    for r, p in enumerate(ranks):
        kk3 = u32(rng.integers(0, 5000, 1000 + 700 * r, dtype=np.uint64).astype(np.uint32))
        if kind == "mixed":
            p.route_phase(kind, kk3, kk3, u8(gen.bernoulli_ops(kk3.numel(), 0.5, 0.2, seed=r)))
        else:
            p.route_phase(kind, kk3)
    for p in ranks:
        p.serve_phase()
    for p in ranks:
        p.finish_phase()
for p in ranks:
    p.close()
hive.gather_ceiling(torch.zeros(64 * 32, dtype=torch.int64, device="cuda"), kk)
torch.cuda.synchronize()
print("ok", t.size(), u.size())
