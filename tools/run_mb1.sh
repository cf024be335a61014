python tools/microbench.py --shapes 4096x4096,11008x4096,4096x11008 --bits 4 --groups 128 --splits 0,1,2,4,8 > gpurun_out/mb1.log 2>&1
python tools/microbench.py --shapes 4096x4096 --bits 4 --groups 128 --splits 0,1,4 --graph >> gpurun_out/mb1.log 2>&1
python tools/microbench.py --shapes 4096x4096 --bits 4 --groups 128 --splits 0 --reps 3 > gpurun_out/mb_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__cluster_dim_y --clock-control none -c 12 --csv --log-file gpurun_out/ncu_launches.csv python tools/microbench.py --shapes 4096x4096 --bits 4 --groups 128 --splits 0 --reps 3 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 5 -c 1 -o gpurun_out/prof_gemv1 python tools/microbench.py --shapes 4096x4096 --bits 4 --groups 128 --splits 0 --reps 3 > gpurun_out/ncu2.log 2>&1
cat gpurun_out/mb1.log
