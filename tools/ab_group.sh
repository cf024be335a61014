set -x
timeout 600 python -m pytest tests -q -m gpu -k "group or batch" 2>&1 | tail -2
for L in old new old new; do echo "== $L"; QIGEN_B200_LIB=build/lib_ab_$L.so timeout 300 python tools/microbench.py --shapes 4096x11008 --bits 2,3,4 --groups 32,128,fc --tokens 1 --graph --group 2>&1 | tail -9; done
