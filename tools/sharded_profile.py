"""Stage timings of the sharded handle at world size 1 (cfg2 step through the
C-ABI collective calls): the library's per-launch CUDA events (hive_profile)
split the step into route, NCCL exchange, owner compaction, the local phase
kernels, result return and unpermute."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
import numpy as np
import torch
import torch.distributed as dist

import gen
from paper_2510_15095_b200 import u32
from paper_2510_15095_b200.sharded import ShardedHive

dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = 1 << 26
ids = np.arange(n, dtype=np.uint32)
keys, vals = u32(gen.keys_of(ids)), u32(gen.vals_of(ids))
qids, _ = gen.mixed_queries(n // 2, n // 2, n, seed=202)
q = u32(gen.keys_of(qids))
dedup = "--dedup" in sys.argv
sh = ShardedHive(gen.CFG2_BUCKETS * 32, batch_max=n, lf_grow=2.0, lf_shrink=0, shard_dedup=dedup)
for rep in range(3):
    if rep == 2:
        sh.table.profile(True)
    sh.table.clear()
    sh.insert(keys, vals)
    sh.find(q)
torch.cuda.synchronize()
p = sh.table.profile_read()
print(json.dumps({"source_dedup": dedup, "ms": {k: round(v[0], 3) for k, v in p.items()},
                  "total_ms": round(sum(v[0] for v in p.values()), 3)}))
sh.close()
dist.destroy_process_group()
