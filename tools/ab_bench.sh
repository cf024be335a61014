# same-box A/B of the bench headline: build/lib_ab_old.so vs build/lib_ab_new.so
for L in old new old new; do
  QIGEN_B200_LIB=build/lib_ab_$L.so timeout 300 python bench.py --steps 200 --warmup 10 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$L', d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
