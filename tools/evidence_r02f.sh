#!/bin/bash
# Final round-2 evidence (one B200), end of the last session: split-aware victim, chained election clears, per-batch prep, paired
# mixed-batch elections: bench line, world-1 sharded lines, launch list + ncu of
# the step kernels, the cfg3 launch list, the step breakdown, the GPU suite.
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build --force > /dev/null
L2="lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum"
ARGS="--steps 1 --warmup 3 --no-secondary --no-cpu-baseline"
python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
tail -c 300 gpurun_out/r02f_bench.json
for ex in nccl p2p; do
  MASTER_PORT=29611 python bench.py --force-sharded --exchange $ex --steps 5 --no-cpu-baseline > gpurun_out/r02f_sharded_$ex.json 2> gpurun_out/r02f_sharded_$ex.err
done
python tools/step_breakdown.py gpurun_out/r02f_step_breakdown.md > gpurun_out/r02f_step_breakdown.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02f_launches.csv python bench.py $ARGS > gpurun_out/r02f_launches_bench.log 2>&1
ncu --set full --metrics $L2 --clock-control none --import-source on \
    -k regex:"k_insert_fast|k_find|k_insert_slow|k_elect_hist|k_elect_scatter" -s 20 -c 5 \
    -o gpurun_out/r02f_prof python bench.py $ARGS > gpurun_out/r02f_prof.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 4000 \
    --log-file gpurun_out/r02f_launches_cfg3.csv python tools/prof_cfg3.py > gpurun_out/r02f_launches_cfg3.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/r02f_pytest_gpu.log 2>&1
tail -3 gpurun_out/r02f_pytest_gpu.log
