"""Run by test_gpu_parity.test_election_modes_over_many_phases in a subprocess (the
election knobs are read once per process): several partitioned-election
batches with heavy duplicates, element-by-element against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gpu_util import Pair  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
n = 1 << 22
p = Pair(-(-(1 << 21) * 100 // (80 * 32)) * 32, lf_grow=2.0, lf_shrink=0)
for rnd in range(5):
    keys = rng.integers(0, 1 << 21, n, dtype=np.uint64).astype(np.uint32)
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    p.insert(keys, vals)
    p.erase(rng.integers(0, 1 << 22, n // 2, dtype=np.uint64).astype(np.uint32))
    if rnd % 2 == 1:                       # a single-table (small) phase in between
        p.insert(keys[: 1 << 16], vals[: 1 << 16] ^ 1)
    p.check_state()
p.find(rng.integers(0, 1 << 22, 1 << 20, dtype=np.uint64).astype(np.uint32))
print("ok")
