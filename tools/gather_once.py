"""One launch of each calibration gather (read-only, + store, + CAS) over a
cfg2-sized block array, for an ncu capture (SURVEY §8(d) ceilings)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
from paper_2510_15095_b200 import hive, u32
nb = gen.CFG2_BUCKETS
blocks = torch.zeros(nb * 32, dtype=torch.int64, device="cuda")
keys = u32(gen.present_keys(1 << 26))
hive.gather_ceiling(blocks, keys)
hive.gather_ceiling_rw(blocks, keys, 1)
hive.gather_ceiling_rw(blocks, keys, 2)
torch.cuda.synchronize()
print("ok")
