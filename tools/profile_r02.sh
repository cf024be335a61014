#!/bin/bash
# Round-2 GPU pass: parity suite, smoke, default bench, ncu launch list + full
# captures (grouped GEMV in the bench, single-config grouped launches for the
# issue-bound 2/3-bit configs, the fused LM head).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
if [ "$1" != "noprep" ]; then
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
fi
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \
    --clock-control none -k 'regex:gemv_group_kernel|group_prep_kernel' -c 6 --csv \
    --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-decode > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_group_kernel -s 1 -c 1 \
    -o gpurun_out/prof_group python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-decode > gpurun_out/ncu_full.log 2>&1
for cfg in "2 fc 4096x11008" "3 fc 4096x11008" "4 128 4096x11008"; do
  set -- $cfg
  ncu --set full --clock-control none --import-source on -k regex:gemv_group_kernel -s 2 -c 1 \
      -o gpurun_out/prof_group_b$1_$2 python tools/microbench.py --group --graph --bits $1 --groups $2 \
      --shapes $3 --reps 2 > gpurun_out/ncu_b$1_$2.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:lm_head_kernel -s 2 -c 1 \
    -o gpurun_out/prof_lmhead python bench.py --workload llama7b --layers 2 --steps 3 --warmup 3 > gpurun_out/ncu_lm.log 2>&1
echo done
