#!/bin/bash
# ncu evidence for the bench (run on the GPU box after `python bench.py` exits 0):
#  1. launch list of the bench command (--metrics gpu__time_duration.sum, no clock
#     control) with DRAM bytes, for the kernel share of a step;
#  2. one `--set full` capture of the dominant kernel (gemv_group_kernel);
#  3. the old per-GEMV path (gemv_kernel) of cfg0 for comparison.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
    --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_group_kernel -s 3 -c 1 \
    -o gpurun_out/prof_group python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
