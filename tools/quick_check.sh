#!/bin/bash
# Quick GPU check after a kernel change: build, the election / mixed parity
# tests, one short bench line (no secondary), cfg4 Zipf.
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build --force > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -k "election or partitioned or duplicates or zipf or ragged_mixed" -m gpu -x -q > gpurun_out/quick_pytest.log 2>&1
tail -1 gpurun_out/quick_pytest.log
timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
timeout 300 python tools/zipf_time.py 2>/dev/null
