"""Sweep the owner-election sizing knobs (HIVE_ELECT_MB / HIVE_ELECT_F /
HIVE_ELECT_JIT) on the bench step: value and per-kernel ms."""
import json, os, subprocess, sys
for spec in sys.argv[1:]:                      # e.g. "MB=32,F=2.5,JIT=0"
    env = dict(os.environ)
    for kv in spec.split(","):
        k, v = kv.split("=")
        env["HIVE_ELECT_" + k] = v
    out = subprocess.run([sys.executable, "bench.py", "--no-cpu-baseline", "--no-secondary", "--steps", "5"],
                         capture_output=True, text=True, env=env).stdout.strip().splitlines()[-1]
    d = json.loads(out)
    k = d["kernels_ms_per_step"]
    print(spec, round(d["value"], 3), round(d["ms_per_step"], 3), round(k.get("k_elect_partition", 0), 3),
          round(k["k_dedup_elect"], 3), round(k.get("elect_clear", 0), 3), round(k.get("k_dedup_resolve", 0), 3),
          round(k["k_insert_fast"], 3), round(k["k_insert_slow"], 3), flush=True)
