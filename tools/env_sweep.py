"""Run the bench step under several environment settings and print value,
ms/step and the per-kernel ms.  Each argument is one setting, e.g.
"HIVE_PREFETCH=0,HIVE_MINB=4" ("-" = no overrides)."""
import json, os, subprocess, sys
for spec in sys.argv[1:]:
    env = dict(os.environ)
    if spec != "-":
        for kv in spec.split(","):
            k, v = kv.split("=")
            env[k] = v
    out = subprocess.run([sys.executable, "bench.py", "--no-cpu-baseline", "--no-secondary", "--steps", "5"],
                         capture_output=True, text=True, env=env).stdout.strip().splitlines()
    if not out:
        print(spec, "FAILED", flush=True)
        continue
    d = json.loads(out[-1])
    k = {n: round(v, 3) for n, v in d["kernels_ms_per_step"].items()}
    print(spec, round(d["value"], 3), round(d["ms_per_step"], 3), json.dumps(k), flush=True)
