"""Does pinned host memory (or big device tensors) slow down VMM growth?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen
from paper_2510_15095_b200 import HiveTable, u8, u32
def cfg3(tag):
    nbat, bsz, U = 32, 1 << 20, 1 << 26
    dev = torch.device("cuda")
    t = HiveTable(1024 * 32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for b in range(nbat):
        ids = gen.uniform_ids(bsz, U, seed=2000 + b)
        k = u32(gen.keys_of(ids)); ops = u8(gen.bernoulli_ops(bsz, 0.4, 0.2, seed=1000 + b))
        torch.cuda.synchronize()
        t.mixed(ops, k, k)
    torch.cuda.synchronize()
    print(tag, "cfg3 half:", round(time.perf_counter() - t0, 3), "s", t.stats()["n_buckets"], flush=True)
cfg3("baseline")
big = torch.empty(6 << 30, dtype=torch.uint8, device="cuda")
cfg3("after 6 GiB device tensor")
pin = [torch.empty(1 << 28, dtype=torch.uint8).pin_memory() for _ in range(5)]
cfg3("after 1.25 GiB pinned host")
