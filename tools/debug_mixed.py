"""Replay test_mixed_grow_and_shrink[7] and report the first divergence in detail."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import gen
from gpu_util import Pair, np8, np32, gpu_dump
from paper_2510_15095_b200 import u8, u32
K = int(sys.argv[1]) if len(sys.argv) > 1 else 7
p = Pair(1024 * 32, resize_k=K)
U = 1 << 17
for b in range(16):
    n = 1 << 14
    ops = gen.bernoulli_ops(n, 0.4, 0.2, seed=1000 + b)
    ids = gen.uniform_ids(n, U, seed=2000 + b)
    keys, vals = gen.keys_of(ids), gen.vals_of(ids ^ b)
    before = p.o.dump_dict()
    sg0, so0 = p.g.stats(), p.o.stats()
    v_g, r_g = p.g.mixed(u8(ops), u32(keys), u32(vals))
    v_g, r_g = np32(v_g), np8(r_g)
    v_o, r_o = p.o.mixed(ops, keys, vals)
    sg, so = p.g.stats(), p.o.stats()
    print(f"batch {b}: before nb g/o {sg0['n_buckets']}/{so0['n_buckets']} after {sg['n_buckets']}/{so['n_buckets']} "
          f"count {sg['count']}/{so['count']} stash g {sg['stash_used']} o {so['stash_live']} grows {sg['grows']}/{so['grows']}")
    bad = np.flatnonzero((r_g != r_o) | (v_g != v_o))
    if len(bad):
        print("  n bad", len(bad), "by op:", np.bincount(ops[bad], minlength=3))
        for i in bad[:8]:
            k = int(keys[i])
            same = np.flatnonzero(keys == keys[i])
            print(f"  i={i} op={ops[i]} key={k:#x} gpu=({r_g[i]},{v_g[i]}) or=({r_o[i]},{v_o[i]}) in_before={k in before}"
                  f" dups={len(same)} ops_of_dups={ops[same].tolist()}")
        dg, do = gpu_dump(p.g), p.o.dump_dict()
        print("  dump sizes", len(dg), len(do), "missing in gpu", len(set(do) - set(dg)), "extra in gpu", len(set(dg) - set(do)))
        break
    dg, do = gpu_dump(p.g), p.o.dump_dict()
    if dg != do:
        print("  dump differs", len(dg), len(do), len(set(do) - set(dg)), len(set(dg) - set(do)))
        break
print("done")
