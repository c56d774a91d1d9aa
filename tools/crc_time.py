"""The cfg2 step on the BitHash pair and on the lookup-based CRC-32 / CRC-64
pair (§V-B; bench.py's secondary `hash_pairs`), alone: insert + find G ops/s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
from paper_2510_15095_b200 import HiveTable, u32

if __name__ == "__main__":
    n = 1 << 26
    dev = torch.device("cuda")
    ids = np.arange(n, dtype=np.uint32)
    keys, vals = u32(gen.keys_of(ids), dev), u32(gen.vals_of(ids), dev)
    qids, _ = gen.mixed_queries(n // 2, n // 2, n, seed=202)
    q = u32(gen.keys_of(qids), dev)
    out = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for hp in ("bithash", "crc"):
        t = HiveTable(gen.CFG2_BUCKETS * 32, lf_grow=2.0, lf_shrink=0, hash=hp)
        res = []
        for rep in range(4):
            t.clear()
            ev[0].record(); t.insert(keys, vals); ev[1].record(); t.find(q); ev[2].record()
            torch.cuda.synchronize()
            if rep:
                res.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
        ins = min(r[0] for r in res); fnd = min(r[1] for r in res)
        out[hp] = {"insert_gops": n / (ins * 1e-3) / 1e9, "find_gops": n / (fnd * 1e-3) / 1e9}
        del t
    print(json.dumps(out), flush=True)
