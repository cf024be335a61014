#!/bin/bash
# Evidence pass for the persistent decode stack: grid-barrier microbenchmark,
# per-phase traces (7B, 65B; with the math off; with barriers' predecessor knobs),
# decode bench lines with and without the stack, ncu launch list of a decode
# step and a full capture of the stack kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
(cd tools/ubench && nvcc -arch=sm_100a -O3 -o gridbar gridbar.cu && timeout 60 ./gridbar) > gpurun_out/gridbar.txt 2>&1
timeout 300 python tools/trace_stack.py 7b 4 > gpurun_out/stack_trace_7b.txt 2>&1
timeout 300 python tools/trace_stack.py 65b 2 > gpurun_out/stack_trace_65b.txt 2>&1
STACK_MODE=1 timeout 300 python tools/trace_stack.py 7b 4 > gpurun_out/stack_trace_7b_nomath.txt 2>&1
timeout 300 python tools/trace_stack.py 7b 4 2 8 1111 > gpurun_out/stack_trace_7b_ksl1111.txt 2>&1
for w in llama7b llama65b; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 5 2>/dev/null | tail -1
  QIGEN_STACK=0 timeout 600 python bench.py --workload $w --steps 50 --warmup 5 2>/dev/null | tail -1
done > gpurun_out/bench_stack.jsonl
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
    --clock-control none -k 'regex:decode_stack_kernel|lm_head_kernel' -s 4 -c 8 --csv \
    --log-file gpurun_out/stack_launches.csv \
    python bench.py --workload llama7b --steps 2 --warmup 3 > gpurun_out/ncu_stack_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_stack -s 2 -c 1 \
    -o gpurun_out/stack7b -f python tools/stack_once.py 7b 8 4 > gpurun_out/ncu_stack.log 2>&1
echo done
