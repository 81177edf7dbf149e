#!/bin/bash
# All BASELINE configs through bench.py (short runs), one JSON line each.
mkdir -p gpurun_out
for c in ternary16384 binary16384 llama4096 llama4096x14336 llama14336x4096 ternary65536 ternary16384b64 ternary4096f32; do
  timeout 900 python bench.py --config $c --steps 500 --warmup 5 --no-cpu > gpurun_out/bench_$c.log 2>&1
  echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print('  ', round(d['value']), d['unit'], 'ms/step', round(d['ms_per_step']*1e3,2), 'us', 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']))
except Exception as e: print('  parse fail', e)"
done
