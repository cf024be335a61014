set -x
timeout 600 python -m pytest tests -m gpu -x -q -k "qgemv or panel" 2>&1 | tail -5
python tools/microbench.py --shapes 4096x4096,11008x4096,4096x11008 --bits 4 --groups 128 --splits 0,1,2,4,8 2>&1
python tools/microbench.py --shapes 4096x4096 --bits 2,3,4 --groups 32,128,fc --splits 0 --graph 2>&1
