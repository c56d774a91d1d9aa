#!/bin/bash
# Round evidence (1 GPU): launch list of the bench command + full ncu captures of
# the hot kernels (one launch each, after the warm-up steps).
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build
ARGS="--steps 1 --warmup 3 --no-secondary --no-cpu-baseline"
# L2 sector / atomic counters are not in --set full on this ncu: add them
L2="lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/launches_bench.log 2>&1
# 5 matching launches per step (hist, scatter, fast, slow, find): skip 4 steps
ncu --set full --metrics $L2 --clock-control none --import-source on \
    -k regex:"k_insert_fast|k_find|k_insert_slow|k_elect_hist|k_elect_scatter" -s 20 -c 5 \
    -o gpurun_out/prof python bench.py $ARGS > gpurun_out/prof_bench.log 2>&1
ncu --set full --metrics $L2 --clock-control none --import-source on -k regex:"k_dedup_elect_part" -s 100 -c 1 \
    -o gpurun_out/prof_elect python bench.py $ARGS > gpurun_out/prof_elect.log 2>&1
python tools/erase_once.py > /dev/null 2>&1
ncu --set full --metrics $L2 --clock-control none --import-source on -k regex:"k_erase" -c 1 \
    -o gpurun_out/prof_erase python tools/erase_once.py > gpurun_out/prof_erase.log 2>&1
ls -la gpurun_out
# config-3 mixed run: per-launch durations of every kernel of the 64 batches
ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 4000 \
    --log-file gpurun_out/launches_cfg3.csv python tools/prof_cfg3.py > gpurun_out/launches_cfg3.log 2>&1
python tools/prof_cfg3.py > gpurun_out/prof_cfg3.json 2>&1
ls -la gpurun_out
