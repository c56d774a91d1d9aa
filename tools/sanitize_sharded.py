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
# hive_load_image: keys placed first-fit in their b1 bucket (64 buckets, split 0), the rest in the stash
from paper_2510_15095_b200 import hive
keys = gen.present_keys(1800)
h1 = hive.hash_keys("bithash1", u32(keys)).cpu().numpy().view(np.uint32)
slots = np.full(64 * 32, np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64)
fill = np.zeros(64, np.int64)
stash = []
for k, h in zip(keys.tolist(), h1.tolist()):
    b = h & 63
    w = np.uint64((k << 32) | k)
    if fill[b] < 32:
        slots[b * 32 + fill[b]] = w
        fill[b] += 1
    else:
        stash.append(w)
u = HiveTable(64 * 32, lf_grow=2.0, lf_shrink=0)
u.load_image(torch.from_numpy(slots.view(np.int64)).cuda(),
             torch.from_numpy(np.array(stash, np.uint64).view(np.int64)).cuda() if stash else None)
v, f = u.find(u32(keys))
assert bool(f.all().item())
torch.cuda.synchronize()
dist.destroy_process_group()
print("ok")
