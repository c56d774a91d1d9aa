"""Config 3: 64 batches x 2^20 mixed ops (40/20/40) over U = 2^26
from 1K buckets with growth and shrink, timed on the device (CUDA events, one
warm-up pass that maps the growth range); PHASED hive_mixed by default,
`--concurrent` for hive_mixed_concurrent.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
from paper_2510_15095_b200 import HiveTable, u8, u32


def main():
    conc = "--concurrent" in sys.argv
    nbat, bsz, U = 64, 1 << 20, 1 << 26
    dev = torch.device("cuda")
    ops = [u8(gen.bernoulli_ops(bsz, 0.4, 0.2, seed=1000 + b), dev) for b in range(nbat)]
    ids = [gen.uniform_ids(bsz, U, seed=2000 + b) for b in range(nbat)]
    ks = [u32(gen.keys_of(i), dev) for i in ids]
    vs = [u32(gen.vals_of(i), dev) for i in ids]
    vo = torch.empty(bsz, dtype=torch.uint32, device=dev)
    rr = torch.empty(bsz, dtype=torch.uint8, device=dev)
    t = HiveTable(1024 * 32)
    run = t.mixed_concurrent if conc else t.mixed
    for b in range(nbat):
        run(ops[b], ks[b], vs[b], vo, rr)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # unprofiled pass first (the per-kernel events of the profiled pass add
    # host work between launches), then the profiled pass for the breakdown
    t.clear()
    torch.cuda.synchronize()
    e0.record()
    for b in range(nbat):
        run(ops[b], ks[b], vs[b], vo, rr)
    e1.record()
    torch.cuda.synchronize()
    ms_noprof = e0.elapsed_time(e1)
    t.clear()
    t.profile(True)
    torch.cuda.synchronize()
    e0.record()
    for b in range(nbat):
        run(ops[b], ks[b], vs[b], vo, rr)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    p = t.profile_read()
    s = t.stats()
    print(json.dumps({"mode": "concurrent" if conc else "phased",
                      "gops": nbat * bsz / (ms_noprof * 1e-3) / 1e9, "ms": ms_noprof,
                      "gops_profiled": nbat * bsz / (ms * 1e-3) / 1e9, "ms_profiled": ms, "kern_ms": {k: round(v[0], 3) for k, v in p.items()},
                      "leftovers": s["leftovers"], "evictions": s["evictions"], "stash_used": s["stash_used"],
                      "n_buckets": s["n_buckets"], "in_b1": s["in_b1"], "count": s["count"]}), flush=True)


if __name__ == "__main__":
    main()
