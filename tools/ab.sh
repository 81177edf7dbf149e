#!/bin/bash
# A/B of an env toggle on the headline bench (cold, rotating index copies) and the warm loop.
#   tools/ab.sh VAR "v1 v2 ..." [config]
var=$1; vals=$2; cfg=${3:-ternary16384}
for v in $vals; do
  for rep in 1 2; do
    env $var=$v timeout 300 python bench.py --config $cfg --steps 1000 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys
d=json.loads(sys.stdin.read()); print('$var=$v', 'cold us', round(d['ms_per_step']*1e3,2), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']))"
  done
  env $var=$v timeout 120 python tools/prof_multiply.py --config $cfg 2>&1 | tail -1
done
