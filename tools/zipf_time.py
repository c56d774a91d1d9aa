"""cfg4 Zipf(0.99) numbers and the paper's imbalanced mix alone (bench.py's
secondary functions), for A/B runs of build / environment options."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

if __name__ == "__main__":
    dev = torch.device("cuda")
    out = {"cfg4_zipf": bench.cfg4_zipf(dev)}
    if "--imbalanced" in sys.argv:
        out["imbalanced"] = bench.imbalanced(dev)
    print(json.dumps(out), flush=True)
