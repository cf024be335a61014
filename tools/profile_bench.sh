#!/bin/bash
# ncu evidence for the bench: launch list (one step = 36 GEMV launches, cold
# cache, serialised) and one full capture of the cfg0 kernel.
set -e
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__cluster_dim_y \
    --clock-control none -k regex:gemv_kernel -s 36 -c 36 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/microbench.py --shapes 4096x4096 --bits 4 --groups 128 --splits 0 --reps 3 > gpurun_out/mb_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 5 -c 1 \
    -o gpurun_out/prof_cfg0 python tools/microbench.py --shapes 4096x4096 --bits 4 --groups 128 --splits 0 --reps 3 > gpurun_out/ncu_full.log 2>&1
echo done
