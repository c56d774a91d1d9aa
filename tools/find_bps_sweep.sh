#!/bin/bash
# k_find persistent-grid residency sweep (HIVE_FIND_BPS blocks per SM) on the cfg2 step.
for b in 3 4 5 6; do
  HIVE_FIND_BPS=$b python bench.py --steps 5 --no-secondary --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'find_blocks_per_sm': $b, 'value': round(d['value'],3), 'lookups_gps': round(d['lookups_gps'],3), 'k_find_ms': round(d['kernels_ms_per_step']['k_find'],3)}))"
done
