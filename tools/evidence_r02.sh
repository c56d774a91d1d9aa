#!/bin/bash
# Round-2 evidence on one B200: the GPU test suite, the bench line, the launch
# list of the bench command, and ncu --set full (+ L2 sector / atomic counters)
# captures of the hot kernels.  Outputs under gpurun_out/ (copied to profiles/).
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build > /dev/null
L2="lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum"
ARGS="--steps 1 --warmup 3 --no-secondary --no-cpu-baseline"
if [ "$1" != "noprof" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py $ARGS > gpurun_out/r02_launches_bench.log 2>&1
# one launch each of the step's kernels after the warm-up steps (6 matching launches per step)
ncu --set full --metrics $L2 --clock-control none --import-source on \
    -k regex:"k_insert_fast|k_find|k_insert_slow|k_elect_hist|k_elect_scatter" -s 20 -c 5 \
    -o gpurun_out/r02_prof python bench.py $ARGS > gpurun_out/r02_prof.log 2>&1
ncu --set full --metrics $L2 --clock-control none --import-source on -k regex:"k_dedup_elect_part" -s 100 -c 1 \
    -o gpurun_out/r02_prof_elect python bench.py $ARGS > gpurun_out/r02_prof_elect.log 2>&1
ncu --set full --metrics $L2 --clock-control none --import-source on -k regex:"k_mixed_mono" -s 70 -c 1 \
    -o gpurun_out/r02_prof_mono python tools/cfg3_time.py --concurrent > gpurun_out/r02_prof_mono.log 2>&1
fi
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
tail -c 400 gpurun_out/r02_bench.json
python -m pytest tests -m gpu -q > gpurun_out/r02_pytest_gpu.log 2>&1
tail -3 gpurun_out/r02_pytest_gpu.log
