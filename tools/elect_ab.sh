#!/bin/bash
# A/B of the owner-election schedule: HIVE_ELECT_SIDE (sub-table clears on a
# side stream) x HIVE_ELECT_FILTER (candidate pre-filter bitmap bits, 0 = off):
# the cfg2 bench step and cfg4 Zipf per setting.  Produced
# profiles/r02b_elect_ab.txt; both options were removed from hive_host.cu /
# hive_kernels.cu after this A/B (neither helped), so the
# settings below now all run the default schedule.
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build > /dev/null || exit 1
for spec in "SIDE=0,FILTER=0" "SIDE=1,FILTER=0" "SIDE=1,FILTER=27" "SIDE=1,FILTER=28" "SIDE=0,FILTER=28"; do
  timeout 300 python tools/elect_sweep.py "$spec" >> gpurun_out/elect_ab.txt 2>&1
  env $(echo $spec | sed 's/SIDE=/HIVE_ELECT_SIDE=/;s/,FILTER=/ HIVE_ELECT_FILTER=/') \
    timeout 300 python tools/zipf_time.py >> gpurun_out/elect_ab.txt 2>&1
done
cat gpurun_out/elect_ab.txt
