import os, sys, subprocess, json
for mb in sys.argv[1:]:
    env = dict(os.environ, HIVE_ELECT_MB=mb)
    out = subprocess.run([sys.executable, "bench.py", "--no-cpu-baseline", "--no-secondary", "--steps", "3"],
                         capture_output=True, text=True, env=env).stdout.strip().splitlines()[-1]
    d = json.loads(out)
    k = d["kernels_ms_per_step"]
    print(mb, round(d["value"], 3), round(k.get("k_elect_partition", 0), 3), round(k["k_dedup_elect"], 3), round(k["k_insert_fast"], 3), flush=True)
