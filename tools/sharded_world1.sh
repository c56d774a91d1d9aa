for ex in nccl p2p; do
  MASTER_PORT=29611 python bench.py --force-sharded --exchange $ex --steps 5 --no-cpu-baseline > gpurun_out/s_$ex.json 2> gpurun_out/s_$ex.err
  MASTER_PORT=29612 python bench.py --cfg5 --cfg5-log2 28 --exchange $ex --steps 3 > gpurun_out/c5_$ex.json 2> gpurun_out/c5_$ex.err
done
for f in s_nccl s_p2p c5_nccl c5_p2p; do grep '^{' gpurun_out/$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['value'],3), round(d['ms_per_step'],3))"; done
