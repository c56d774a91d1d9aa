#!/bin/bash
# cfg3 (64 x 2^20-op mixed batches) vs the lanes-per-op of each probe kernel:
# the small batches are latency-bound, where fewer lanes per op means more ops
# in flight.  One line per setting: G_INSERT/G_FIND/G_ERASE/G_SLOW, G ops/s,
# per-kernel ms.
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build > /dev/null || exit 1
for spec in "4 4 2 2" "2 2 2 2" "2 4 2 2" "4 2 2 2" "4 4 1 2" "4 4 2 1" "2 2 1 1" "8 8 4 4"; do
  set -- $spec
  out=$(HIVE_G_INSERT=$1 HIVE_G_FIND=$2 HIVE_G_ERASE=$3 HIVE_G_SLOW=$4 timeout 300 python tools/cfg3_time.py 2>/dev/null)
  echo "G $spec :: $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['gops'],3), d['kern_ms'])")" >> gpurun_out/cfg3_g_sweep.txt
done
cat gpurun_out/cfg3_g_sweep.txt
