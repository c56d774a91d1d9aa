#!/bin/bash
# Step-3 victim choice A/B (-DHIVE_VICTIM_LOOK=v: the first of v slots whose
# resident's other bucket is split; 0 = rotating slot): cfg3, the cfg2 step,
# and the Step-3 parity tests at v = 4.
mkdir -p gpurun_out
for v in 0 2 4 8 16; do
  HIVE_NVCC_DEFINES="-DHIVE_VICTIM_LOOK=$v" python -m paper_2510_15095_b200.build --force > /dev/null || exit 1
  c3=$(timeout 300 python tools/cfg3_time.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['gops'],3), d['kern_ms']['k_insert_slow'], d['kern_ms'].get('k_insert_slow(reinsert)'), d['evictions'], d['leftovers'], d['stash_used'])")
  c2=$(timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print(round(d['value'],3), round(k['k_insert_slow'],3))")
  echo "VICTIM_LOOK=$v cfg3: $c3 | cfg2: $c2" >> gpurun_out/victim_ab.txt
  if [ $v = 4 ]; then
    timeout 900 python -m pytest tests/test_gpu_parity.py -k "high_load or grow_and_shrink or zipf or overflow or ragged_mixed" -m gpu -x -q > gpurun_out/victim_pytest.log 2>&1
    tail -1 gpurun_out/victim_pytest.log >> gpurun_out/victim_ab.txt
  fi
done
python -m paper_2510_15095_b200.build --force > /dev/null
cat gpurun_out/victim_ab.txt
