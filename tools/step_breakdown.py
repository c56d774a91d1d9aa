"""Insertion step breakdown vs load factor (Fig. insertion_breakdown;
SURVEY §8(f) NEXT-2).  A table of NB buckets (growth off) is filled in batches
that raise LF from 0.55 to 0.97.  For each batch the insert kernels run in
their clock64-instrumented form (hive_profile level 2): per warp region, the
max-over-lanes end minus the min-over-lanes start clock, summed
into Step 1 (replace), Step 2 (claim-and-commit), Step 3 (bounded eviction)
and Step 4 (stash fallback).  Shares are of the four-step total, as in the
paper's figure; kernel times (CUDA events) and step outcome counters are
reported beside them.

`python tools/step_breakdown.py [out.md] [--log2-buckets B]`"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
from paper_2510_15095_b200 import HiveTable, u32

POINTS = [0.55, 0.60, 0.65, 0.70, 0.75, 0.80, 0.85, 0.88, 0.90, 0.92, 0.94, 0.95, 0.96, 0.97]


def breakdown(nb: int, points=POINTS):
    slots = nb * 32
    t = HiveTable(slots, lf_grow=2.0, lf_shrink=0, keys_unique=True)
    ids = np.arange(int(points[-1] * slots) + 1, dtype=np.uint32)
    keys, vals = u32(gen.keys_of(ids)), u32(gen.vals_of(ids))
    lo = int(points[0] * slots)
    t.insert(keys[:lo], vals[:lo])
    rows = []
    prev = t.stats()
    for lf in points[1:]:
        hi = int(lf * slots)
        t.profile(2)
        t.insert(keys[lo:hi], vals[lo:hi])
        torch.cuda.synchronize()
        p = t.profile_read()
        t.profile(False)
        s = t.stats()
        cyc = [a - b for a, b in zip(s["step_cycles"], prev["step_cycles"])]
        tot = max(1, sum(cyc))
        d = {k: s[k] - prev[k] for k in ("count", "step3", "stash_pushes", "leftovers", "evictions")}
        rows.append({"lf_from": round(lo / slots, 3), "lf_to": lf, "n": hi - lo,
                     "share": [c / tot for c in cyc], "cycles": cyc,
                     "ms_fast": p.get("k_insert_fast", (0.0, 0))[0], "ms_slow": p.get("k_insert_slow", (0.0, 0))[0],
                     "placed_step2": d["count"] - d["leftovers"], "placed_step3": d["step3"],
                     "stashed": d["stash_pushes"], "leftovers": d["leftovers"], "evictions": d["evictions"],
                     "stash_used": s["stash_used"]})
        prev, lo = s, hi
    t.close()
    return rows


def main():
    args = sys.argv[1:]
    log2 = 20
    if "--log2-buckets" in args:
        i = args.index("--log2-buckets")
        log2 = int(args[i + 1])
        del args[i:i + 2]
    out_md = args[0] if args else None
    rows = breakdown(1 << log2)
    for r in rows:
        print(json.dumps(r), flush=True)
    if out_md:
        with open(out_md, "w") as f:
            f.write(f"# Insertion step breakdown vs load factor (B200, 2^{log2} buckets, keys unique)\n\n")
            f.write("Method (PAPER:634): clock64() per warp region, max-over-lanes end minus min-over-lanes "
                    "start, summed over warps (hive_profile level 2, `tools/step_breakdown.py`).  Step 1 = "
                    "replace probe (b1, spill-filtered b2, stash), Step 2 = claim-and-commit (k_insert_fast); "
                    "Step 3 = bounded eviction rounds, Step 4 = stash push (k_insert_slow).  Paper (RTX 4090, "
                    "PAPER:636): Steps 1-2 > 95% at LF 0.55-0.75, Step 3 0.02-2.2%, Step 4 ~41% at 0.97.\n\n")
            f.write("| LF batch | ops | Step 1 | Step 2 | Step 3 | Step 4 | Steps 1-2 | fast ms | slow ms | "
                    "placed by claim | by eviction | stashed | evictions |\n"
                    "|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                sh = r["share"]
                f.write(f"| {r['lf_from']:.2f}-{r['lf_to']:.2f} | {r['n']} | {100 * sh[0]:.1f}% | "
                        f"{100 * sh[1]:.1f}% | {100 * sh[2]:.2f}% | {100 * sh[3]:.2f}% | "
                        f"{100 * (sh[0] + sh[1]):.1f}% | {r['ms_fast']:.3f} | {r['ms_slow']:.3f} | "
                        f"{r['placed_step2']} | {r['placed_step3']} | {r['stashed']} | {r['evictions']} |\n")


if __name__ == "__main__":
    main()
