#!/bin/bash
# Step-3 kernel residency A/B (HIVE_MINB_SLOW: min resident blocks per SM of
# k_insert_slow = its register cap): cfg2 step (k_insert_slow ms) and cfg3.
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build > /dev/null || exit 1
for m in 4 5 6 1; do
  echo "MINB_SLOW=$m" >> gpurun_out/slow_ab.txt
  HIVE_MINB_SLOW=$m timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 5 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],3), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})" >> gpurun_out/slow_ab.txt
  HIVE_MINB_SLOW=$m timeout 300 python tools/cfg3_time.py 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['gops'],3), d['kern_ms']['k_insert_slow'])" >> gpurun_out/slow_ab.txt
done
cat gpurun_out/slow_ab.txt
