"""Experiment: does partitioning a large insert / find phase by
b1 range into L2-sized slices cut DRAM traffic and time?  The table and batch
are cfg2's (2^26 keys, 2,207,529 buckets).  The batch is reordered on the GPU
by a stable sort on the slice id floor(b1 * P / n_b) (ops keep their relative
order inside a slice), then the unmodified hive_insert / hive_find kernels run
on the reordered batch.  Prints one JSON line per configuration."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_2510_15095_b200 import HiveTable, hive, u32  # noqa: E402


def b1_of(keys, m, split):
    h = hive.hash_keys("bithash1", keys).to(torch.int64) & 0xFFFFFFFF
    mask = (1 << m) - 1
    b = h & mask
    return torch.where(b < split, h & (2 * mask + 1), b)


def timed(fn, reps=3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return min(ts)


def main():
    dev = torch.device("cuda")
    n = 1 << 26
    nb = gen.CFG2_BUCKETS
    m, split = 21, nb - (1 << 21)
    ids = np.arange(n, dtype=np.uint32)
    keys, vals = u32(gen.keys_of(ids), dev), u32(gen.vals_of(ids), dev)
    qids, _ = gen.mixed_queries(n // 2, n // 2, n, seed=202)
    q = u32(gen.keys_of(qids), dev)
    for unique in (True, False):
        t = HiveTable(nb * 32, lf_grow=2.0, lf_shrink=0, keys_unique=unique)
        vo = torch.empty(n, dtype=torch.uint32, device=dev)
        fo = torch.empty(n, dtype=torch.uint8, device=dev)
        st = torch.empty(n, dtype=torch.uint8, device=dev)
        kb1, qb1 = b1_of(keys, m, split), b1_of(q, m, split)
        for P in (1, 8, 16, 32, 64, 128, 256):
            if P == 1:
                kp, vp, qp = keys, vals, q
            else:
                ks = torch.sort(kb1 * P // nb, stable=True).indices
                qs = torch.sort(qb1 * P // nb, stable=True).indices
                i32 = lambda x, ix: x.view(torch.int32)[ix].contiguous().view(torch.uint32)
                kp, vp, qp = i32(keys, ks), i32(vals, ks), i32(q, qs)

            def ins():
                t.insert(kp, vp, st)

            def clear_ins():
                t.clear()
                ins()
            # insert time: clear outside the timed region
            tins = []
            for _ in range(3):
                t.clear()
                tins.append(timed(ins, 1))
            tf = timed(lambda: t.find(qp, vo, fo))
            hits = int(fo.sum().item())
            s = t.stats()
            print(json.dumps({"unique": unique, "P": P, "insert_ms": min(tins), "find_ms": tf,
                              "hits": hits, "leftovers": s["leftovers"], "evictions": s["evictions"],
                              "stash": s["stash_used"]}), flush=True)
        # cost of the unpermute gathers that a sliced phase would add
        perm = torch.randperm(n, device=dev)
        g4 = timed(lambda: vo.view(torch.int32)[perm])
        g1 = timed(lambda: fo[perm])
        print(json.dumps({"gather_u32_ms": g4, "gather_u8_ms": g1}), flush=True)
        t.close()


if __name__ == "__main__":
    main()
