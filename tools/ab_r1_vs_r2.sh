cd ab_r1 && for i in 1 2; do python bench.py --steps 5 --no-secondary --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R1', round(d['value'],3), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"; done; cd ..
for i in 1 2; do python bench.py --steps 5 --no-secondary --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R2', round(d['value'],3), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"; done
python tools/cfg3_time.py --concurrent
python -m pytest tests/test_gpu_concurrent.py -q -x 2>&1 | tail -2
