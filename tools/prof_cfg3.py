"""Per-batch wall time and per-kernel device time of the config-3 mixed run."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen
from paper_2510_15095_b200 import HiveTable, u8, u32
nbat, bsz, U = 64, 1 << 20, 1 << 26
dev = torch.device("cuda")
ops = [u8(gen.bernoulli_ops(bsz, 0.4, 0.2, seed=1000 + b), dev) for b in range(nbat)]
ids = [gen.uniform_ids(bsz, U, seed=2000 + b) for b in range(nbat)]
ks = [u32(gen.keys_of(i), dev) for i in ids]
vs = [u32(gen.vals_of(i), dev) for i in ids]
vo = torch.empty(bsz, dtype=torch.uint32, device=dev)
rr = torch.empty(bsz, dtype=torch.uint8, device=dev)
if len(sys.argv) > 1:   # reproduce the bench state: a big table + its scratch first
    big = HiveTable(gen.CFG2_BUCKETS * 32, lf_grow=2.0, lf_shrink=0)
    n = 1 << 26
    kk = u32(gen.keys_of(np.arange(n, dtype=np.uint32)), dev)
    big.insert(kk, kk); big.find(kk); torch.cuda.synchronize()
    if sys.argv[1] == "del":
        del big
    torch.cuda.synchronize()
t = HiveTable(1024 * 32)
t.profile(True)
torch.cuda.synchronize()
walls = []
t0 = time.perf_counter()
for b in range(nbat):
    a = time.perf_counter()
    t.mixed(ops[b], ks[b], vs[b], vo, rr)
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - a)
tot = time.perf_counter() - t0
p = t.profile_read()
print(json.dumps({"total_s": tot, "walls_ms": [round(w * 1e3, 2) for w in walls],
                  "kern_ms": {k: round(v[0], 3) for k, v in p.items()},
                  "launches": {k: v[1] for k, v in p.items()}, "stats": t.stats()}))
