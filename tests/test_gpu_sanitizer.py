"""The small workload that touches every kernel family, run as a
plain subprocess.  compute-sanitizer (memcheck / racecheck / synccheck) is
closed on this GPU pool since late round 2, so the workloads run without it
here; their last sanitizer-clean runs (memcheck, racecheck and synccheck over
tools/sanitize_run.py, memcheck over tools/sanitize_sharded.py) are recorded in
profiles/r02_pytest_gpu.log.  Each script checks its results against the
oracle and prints "ok"."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("script", ["sanitize_run.py", "sanitize_sharded.py"])
def test_every_kernel_family_workload(script):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", script)], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "ok" in r.stdout
