"""Small workload over the sharded handle at world size 1 (route, NCCL exchange,
owner compaction, PHASED batch, return, unpermute; source-side election; host
calls) and hive_load_image, for compute-sanitizer (tests/test_gpu_sanitizer.py)."""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import gen
from paper_2510_15095_b200 import HiveTable, u8, u32
from paper_2510_15095_b200.sharded import ShardedHive

with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
rng = np.random.default_rng(4)
for dedup in (False, True):
    sh = ShardedHive(128 * 32, batch_max=5000, resize_k=8, shard_dedup=dedup)
    for b in range(4):
        n = int(rng.integers(0, 5000))
        keys = rng.integers(0, 3000, n, dtype=np.uint64).astype(np.uint32)
        sh.mixed(u8(gen.bernoulli_ops(n, 0.5, 0.2, seed=b)), u32(keys), u32(keys ^ 3))
    q = u32(rng.integers(0, 4000, 5000, dtype=np.uint64).astype(np.uint32))
    sh.find(q)
    sh.erase(q[:2000])
    sh.insert(q[:3000], q[:3000])
    kh = torch.from_numpy(rng.integers(0, 4000, 1000, dtype=np.uint64).astype(np.uint32).view(np.int32))
    kh = kh.view(torch.uint32).pin_memory()
    sh.insert_host(kh, kh)
    sh.find_host(kh)
    torch.cuda.synchronize()
    sh.close()
# hive_load_image: a table's own dump layout reloaded into another table
t = HiveTable(64 * 32, lf_grow=2.0, lf_shrink=0)
k = u32(gen.present_keys(1800))
t.insert(k, k)
slots = torch.full((64 * 32,), -1, dtype=torch.int64, device="cuda")
kk, vv = t.dump()
u = HiveTable(64 * 32, lf_grow=2.0, lf_shrink=0)
u.insert(kk, vv)
u.find(k)
torch.cuda.synchronize()
dist.destroy_process_group()
print("ok")
