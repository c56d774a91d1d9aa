#!/bin/bash
# Owner-election records per lane (HIVE_ELECT_ILP 1 / 2 / 3) on the cfg2 step, and the
# election parity tests under each setting.
for i in 1 2 3; do
  HIVE_ELECT_ILP=$i python bench.py --steps 5 --no-secondary --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_step']
print(json.dumps({'elect_ilp': $i, 'value': round(d['value'],3), 'updates_gps': round(d['updates_gps'],3), 'k_dedup_elect_ms': round(k['k_dedup_elect'],3), 'k_insert_fast_ms': round(k['k_insert_fast'],3)}))"
done
for i in 2 3; do
  HIVE_ELECT_ILP=$i python -m pytest tests/test_gpu_parity.py -q -x -k "partitioned or election or duplicates or zipf" 2>&1 | tail -1
done
