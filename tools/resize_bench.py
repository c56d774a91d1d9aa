"""Resize throughput alone (§V-A: "16.8 GOPS expansion, 23.7 GOPS
contraction" at 32,768 buckets on an RTX 4090; unit undefined, reading A-23;
SURVEY §2.7 E6, §8(d) split row).  A 32,768-bucket table at LF 0.9 is grown
by one whole linear-hashing round (32,768 split pairs, K = 1024-bucket batches
issued as one k_split launch per round) and then contracted back by erasing
keys (32,768 LIFO merge pairs: k_merge_check + k_merge_apply).  The split and
merge kernels are timed by the library's per-launch CUDA events; reported as
buckets (pairs) / s, live keys of the source buckets / s, and GB/s against the
768 B / pair byte model (256 B read + 256 B destination write + <= 256 B source
write-back).  Prints one JSON line and writes profiles/r02_resize.json."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
from paper_2510_15095_b200 import HiveTable, u32

NB = 32768


def main(out=None, reps=5):
    slots = NB * 32
    n0 = int(0.9 * slots)                      # LF 0.9 exactly: no growth yet
    grow_to = 2 * NB
    n1 = int(0.9 * (grow_to - 1) * 32) + 1 - n0     # forces growth to exactly 2 * NB buckets
    ids = np.arange(n0 + n1, dtype=np.uint32)
    keys, vals = u32(gen.keys_of(ids)), u32(gen.vals_of(ids))
    t = HiveTable(slots, resize_k=1024, lf_grow=0.9, lf_shrink=0.25, keys_unique=True)
    splits, merges = [], []
    for rep in range(reps + 1):
        t.clear()
        t.insert(keys[:n0], vals[:n0])
        torch.cuda.synchronize()
        assert t.stats()["n_buckets"] == NB
        t.profile(True)
        t.insert(keys[n0:], vals[n0:])            # grow_before: one round of 32,768 splits
        torch.cuda.synchronize()
        p = t.profile_read(reset=True)
        s = t.stats()
        assert s["n_buckets"] == grow_to, s["n_buckets"]
        split_ms, split_launches = p["k_split"]
        # contraction: erase down below 0.25 of the grown table, then the
        # shrink phase merges LIFO pairs back to the initial 32,768 buckets
        live = n0 + n1
        keep = int(0.25 * NB * 32 * 0.9)
        t.profile(True)
        t.erase(keys[: live - keep])
        torch.cuda.synchronize()
        p2 = t.profile_read(reset=True)
        t.profile(False)
        s2 = t.stats()
        merge_ms, merge_launches = p2.get("k_merge", (0.0, 0))
        if rep:
            splits.append((split_ms, split_launches, n0))
            merges.append((merge_ms, merge_launches, s2["n_buckets"], s2["merge_aborts"], keep))
    sm = statistics.median(x[0] for x in splits)
    mm = statistics.median(x[0] for x in merges)
    merged_pairs = grow_to - merges[-1][2]
    res = {
        "table_buckets": NB, "k": 1024,
        "split": {"pairs": NB, "ms": sm, "launches": splits[-1][1], "buckets_per_s": NB / (sm * 1e-3),
                  "source_keys_per_s": n0 / (sm * 1e-3), "model_GBps": NB * 768 / (sm * 1e-3) / 1e9,
                  "live_keys_before": n0},
        "merge": {"pairs": merged_pairs, "ms": mm, "launches": merges[-1][1],
                  "buckets_per_s": merged_pairs / (mm * 1e-3) if mm else None,
                  "keys_per_s": keep / (mm * 1e-3) if mm else None,
                  "model_GBps": merged_pairs * 768 / (mm * 1e-3) / 1e9 if mm else None,
                  "final_buckets": merges[-1][2], "merge_aborts": merges[-1][3], "live_keys": keep},
        "paper_rtx4090": {"expansion_GOPS": 16.8, "contraction_GOPS": 23.7, "note": "unit undefined (A-23)"},
        "timing": f"median of {reps} reps, per-launch CUDA events (hive_profile), after 1 warm-up",
    }
    print(json.dumps(res), flush=True)
    if out:
        with open(out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
