#!/bin/bash
# A/B of library builds on the headline bench: tools/ab_lib.sh <lib1> <lib2> ... [config via CFG]
cfg=${CFG:-ternary16384}
for L in "$@"; do
  for rep in 1 2; do
    RSR_BENCH_NO_E2E=1 RSR_B200_LIB=$L timeout 300 python bench.py --config $cfg --steps 1000 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); print('$L', 'cold us', round(d['ms_per_step']*1e3,2), 'frac', round(d['roofline']['frac'],3))"
  done
  RSR_B200_LIB=$L timeout 120 python tools/prof_multiply.py --config $cfg 2>&1 | tail -1
done
