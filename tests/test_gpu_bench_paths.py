"""bench.py's sharded and config-5 paths stay runnable (small sizes, world
size 1): each prints one JSON line whose correctness guards passed."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
def test_bench_sharded_world1(exchange):
    d = _run(["--force-sharded", "--exchange", exchange, "--n-log2", "20", "--steps", "2", "--no-cpu-baseline"])
    assert d["value"] > 0 and d["n_gpus"] == 1 and "hash-sharded" in d["config"]["parallelism"]


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
def test_bench_cfg5_small(exchange):
    d = _run(["--cfg5", "--cfg5-log2", "22", "--exchange", exchange, "--steps", "1"])
    assert d["value"] > 0 and d["scaling"] == "strong" and d["count_total"] == (1 << 22) - (1 << 19)
