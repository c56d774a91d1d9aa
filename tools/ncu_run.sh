#!/bin/bash
# Round evidence (1 GPU): launch list of the bench command + one full ncu capture of the hot kernels.
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build
ARGS="--steps 1 --warmup 1 --no-secondary --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_insert_fast|k_find|k_dedup_elect_part|k_insert_slow|k_elect_hist|k_elect_scatter" -s 40 -c 12 \
    -o gpurun_out/prof python bench.py $ARGS > gpurun_out/prof_bench.log 2>&1
python tools/erase_once.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_erase" -c 1 \
    -o gpurun_out/prof_erase python tools/erase_once.py > gpurun_out/prof_erase.log 2>&1
ls -la gpurun_out
