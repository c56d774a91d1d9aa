#!/bin/bash
# Last check of the final code on one B200: the bench line, smoke(), the GPU suite.
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build --force > /dev/null
python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
tail -c 300 gpurun_out/r02g_bench.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; tail -1 gpurun_out/r02g_smoke.log
python -m pytest tests -m gpu -q > gpurun_out/r02g_pytest_gpu.log 2>&1
tail -3 gpurun_out/r02g_pytest_gpu.log
