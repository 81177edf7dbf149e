#!/bin/bash
# A/B of the bench's launch mode (independent stream vs dependent chain): tools/launch_ab.sh configs...
for rep in 1 2; do for c in "$@"; do for mode in independent dependent; do
  timeout 300 python bench.py --config $c --no-cpu --steps 400 --launch $mode 2>/tmp/launch_ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', '$mode', round(d['ms_per_step']*1e3,3), 'us', 'frac', round(d['roofline']['frac'],3))" || tail -3 /tmp/launch_ab.err
done; done; done
