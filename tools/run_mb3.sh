timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python tools/microbench.py --shapes 4096x4096,11008x4096,4096x11008 --bits 4 --groups 128 --splits 0,2,4,8 2>&1
python tools/microbench.py --shapes 4096x4096 --bits 2,3,4 --groups 32,128,fc --splits 0 --graph 2>&1
python tools/microbench.py --shapes 4096x4096 --bits 4 --groups 128 --splits 0 --reps 3 > gpurun_out/mb_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 5 -c 1 -o gpurun_out/prof_gemv3 python tools/microbench.py --shapes 4096x4096 --bits 4 --groups 128 --splits 0 --reps 3 > gpurun_out/ncu3.log 2>&1
echo ncu=$?
