#!/bin/bash
# Thresholded two-choice placement sweep (reading A-21): rebuild
# libhive.so with -DHIVE_TWO_CHOICE_T=T and time the cfg2 step and cfg3.
mkdir -p gpurun_out
for T in "$@"; do
  HIVE_NVCC_DEFINES="-DHIVE_TWO_CHOICE_T=$T" python -m paper_2510_15095_b200.build --force > /dev/null
  python bench.py --steps 5 --no-secondary --no-cpu-baseline > gpurun_out/tc$T.json 2> gpurun_out/tc$T.err
  python tools/cfg3_time.py > gpurun_out/tc3_$T.json 2>> gpurun_out/tc$T.err
  python - "$T" <<'PY'
import json, sys
T = sys.argv[1]
d = json.loads([l for l in open(f"gpurun_out/tc{T}.json") if l.startswith("{")][-1])
c = json.loads([l for l in open(f"gpurun_out/tc3_{T}.json") if l.startswith("{")][-1])
k = d["kernels_ms_per_step"]
print(json.dumps({"two_choice_t": int(T), "cfg2_value": round(d["value"], 3), "updates": round(d["updates_gps"], 3),
                  "lookups": round(d["lookups_gps"], 3), "p_h1": round(d["roofline"]["p_h1"], 4),
                  "kern": {n: round(v, 3) for n, v in k.items()}, "cfg2_leftovers": d["table_stats"]["leftovers"],
                  "cfg3_gops": round(c["gops"], 3), "cfg3_kern": c["kern_ms"], "cfg3_leftovers": c["leftovers"]}))
PY
done
python -m paper_2510_15095_b200.build --force > /dev/null
