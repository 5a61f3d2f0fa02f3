#!/bin/bash
# Runs bench.py against each experimental library under variants/ (kernel-shape sweep).
for d in variants/*/; do
  n=$(basename $d)
  v=$(MCB_LIB=$d/libmcb.so timeout 120 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-clocks --no-configs 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('%.4g samples/s  %.2f ms/step  frac %.3f' % (j['value'], j['ms_per_step'], j['roofline']['frac']))")
  echo "$n: $v"
done
