#!/bin/bash
# ncu --set full of the cfg3 probe kernels at a late batch (table ~0.6 M
# buckets): what bounds the 2^20-op batch kernels.
mkdir -p gpurun_out
python -m paper_2510_15095_b200.build > /dev/null || exit 1
L2="lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_atom.sum"
ncu --set full --metrics $L2 --clock-control none --import-source on \
    -k regex:"k_insert_fast|k_insert_slow|k_find|k_erase|k_dedup_elect" -s 230 -c 6 \
    -o gpurun_out/r02d_cfg3_prof python tools/prof_cfg3.py > gpurun_out/r02d_cfg3_prof.log 2>&1
tail -3 gpurun_out/r02d_cfg3_prof.log
