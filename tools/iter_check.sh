#!/bin/bash
# One iteration on the B200: rebuild, election micro-benchmark, cfg3 timing,
# and the mixed-path parity tests.
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build > /dev/null || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/elect_micro tools/elect_micro.cu && \
  timeout 300 /tmp/elect_micro > gpurun_out/elect_micro.txt 2>&1
timeout 600 python tools/cfg3_time.py > gpurun_out/cfg3_time.json 2> gpurun_out/cfg3_time.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullscale.py tests/test_gpu_sanitizer.py tests/test_gpu_concurrent.py -m gpu -x -q > gpurun_out/iter_pytest.log 2>&1
tail -3 gpurun_out/iter_pytest.log
cat gpurun_out/cfg3_time.json
