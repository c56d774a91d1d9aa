#!/bin/bash
# A/B of the optimistic claim placement (-DHIVE_CLAIM_ROT=0 / 1 / 2, a rebuild
# each) on the cfg2 bench step: insert-phase time, kernel times, leftovers.
mkdir -p gpurun_out
for r in 0 1 2; do
  HIVE_NVCC_DEFINES="-DHIVE_CLAIM_ROT=$r" python -m paper_2510_15095_b200.build --force > /dev/null
  python bench.py --steps 5 --no-secondary --no-cpu-baseline > gpurun_out/rot$r.json 2>gpurun_out/rot$r.err
  python - "$r" <<'PY'
import json, sys
r = sys.argv[1]
d = json.loads([l for l in open(f"gpurun_out/rot{r}.json") if l.startswith("{")][-1])
k = d["kernels_ms_per_step"]
print(json.dumps({"rot": int(r), "value": round(d["value"], 3), "updates": round(d["updates_gps"], 3),
                  "lookups": round(d["lookups_gps"], 3), "fast_ms": round(k["k_insert_fast"], 3),
                  "slow_ms": round(k["k_insert_slow"], 3), "leftovers": d["table_stats"]["leftovers"],
                  "evictions": d["table_stats"]["evictions"]}))
PY
done
python -m paper_2510_15095_b200.build --force > /dev/null
