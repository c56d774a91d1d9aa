"""compute-sanitizer memcheck / racecheck / synccheck over a small workload that
touches every kernel family."""
import os
import shutil
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,script", [("memcheck", "sanitize_run.py"), ("racecheck", "sanitize_run.py"),
                                         ("synccheck", "sanitize_run.py"), ("memcheck", "sanitize_sharded.py")])
def test_compute_sanitizer(tool, script):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "17", "--print-limit", "20",
           sys.executable, os.path.join(ROOT, "tools", script)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "ok" in r.stdout
