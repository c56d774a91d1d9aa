import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen
from paper_2510_15095_b200 import HiveTable, u32
n = int(sys.argv[1]); uniq = sys.argv[2] == "1"
t = HiveTable(1 << 20, lf_grow=2.0, lf_shrink=0, keys_unique=uniq)
k = gen.present_keys(n)
st = t.insert(u32(k), u32(k))
torch.cuda.synchronize()
print("G", os.environ.get("HIVE_G_INSERT"), "n", n, "uniq", uniq, "ok", t.stats()["count"], flush=True)
