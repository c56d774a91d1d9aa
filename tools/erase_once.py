"""One cfg2-scale erase of 2^25 present keys (for an ncu capture of k_erase)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen
from paper_2510_15095_b200 import HiveTable, u32
n = 1 << 26
t = HiveTable(gen.CFG2_BUCKETS * 32, lf_grow=2.0, lf_shrink=0)
ids = np.arange(n, dtype=np.uint32)
k = u32(gen.keys_of(ids))
t.insert(k, u32(gen.vals_of(ids)))
e = t.erase(k[: n // 2])
torch.cuda.synchronize()
print(int(e.sum()))
