#!/bin/bash
# A/B: each election part's sub-table cleared by a memset between launches
# (HIVE_ELECT_CHAIN=0) or by the previous part's launch in its tail (=1):
# the cfg2 bench step (3 runs each) and cfg4 Zipf, plus the election parity
# tests with the chain on.
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build > /dev/null || exit 1
for rep in 1 2 3; do
  for c in 0 1; do
    timeout 300 python tools/elect_sweep.py "CHAIN=$c" >> gpurun_out/elect_chain_ab.txt 2>&1
  done
done
for c in 0 1; do
  echo "CHAIN=$c $(HIVE_ELECT_CHAIN=$c timeout 300 python tools/zipf_time.py)" >> gpurun_out/elect_chain_ab.txt 2>&1
done
HIVE_ELECT_CHAIN=1 timeout 900 python -m pytest tests/test_gpu_parity.py -k "election or partitioned or split_geometry" -m gpu -x -q > gpurun_out/elect_chain_pytest.log 2>&1
tail -1 gpurun_out/elect_chain_pytest.log >> gpurun_out/elect_chain_ab.txt
cat gpurun_out/elect_chain_ab.txt
