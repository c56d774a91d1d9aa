"""CSR sweep of Fig. 4 on the GPU: Collision Speedup Ratio
E[Y] / Y_observed for BitHash1, BitHash2, CRC-32 and CRC-64 over m = 512^2
single-slot bins, n = 512 ... 2048^2, with two key sets: distinct random keys
(the workload generator) and sequential keys 0..n-1.  Y comes from
hive_collisions (device bitmap); E[Y] is Theorem 1's closed form.

    python tools/csr_sweep.py [out.md]
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_2510_15095_b200 import hive, u32  # noqa: E402


def expected(n, m):
    return n - m * (1.0 - math.exp(n * math.log1p(-1.0 / m)))


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    m = 512 * 512
    ns = [512 << (2 * i) for i in range(7)]           # 512 ... 2^21 ... 2048^2 = 2^22
    ns = [n for n in ns if n <= 2048 * 2048] + ([2048 * 2048] if 2048 * 2048 not in ns else [])
    fns = ["bithash1", "bithash2", "crc32", "crc64"]
    lines = ["| keys | n | E[Y] | " + " | ".join(f"CSR {f}" for f in fns) + " |",
             "|---|---:|---:|" + "---:|" * len(fns)]
    for kind in ("random", "sequential"):
        for n in ns:
            keys = gen.present_keys(n) if kind == "random" else np.arange(n, dtype=np.uint32)
            d = u32(keys)
            ey = expected(n, m)
            row = []
            for f in fns:
                y = hive.collisions(f, d, m)
                row.append(f"{ey / y:.4f}" if y else "inf")
            lines.append(f"| {kind} | {n} | {ey:.1f} | " + " | ".join(row) + " |")
    txt = "\n".join(lines)
    print(txt)
    if out:
        with open(out, "w") as fh:
            fh.write(f"# CSR sweep (Fig. 4 setup, m = 512^2 bins) on {torch.cuda.get_device_name()}\n\n")
            fh.write(txt + "\n")


if __name__ == "__main__":
    main()
