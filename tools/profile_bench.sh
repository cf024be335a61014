#!/bin/bash
# ncu evidence for the bench (run on the GPU box after `python bench.py` exits 0):
#  1. launch list of the step's kernels (--metrics gpu__time_duration.sum and DRAM
#     bytes, no clock control): activation prep + grouped GEMV;
#  2. one `--set full` capture of the dominant kernel (gemv_group_kernel).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
    --clock-control none -k 'regex:gemv_group_kernel|group_prep_kernel' -c 6 --csv \
    --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_group_kernel -s 1 -c 1 \
    -o gpurun_out/prof_group python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
