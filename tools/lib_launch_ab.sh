#!/bin/bash
# A/B of library builds x bench launch modes: tools/lib_launch_ab.sh "<lib list>" configs...  ("-" = current)
libs=$1; shift
for rep in 1 2; do for c in "$@"; do for lib in $libs; do for mode in independent dependent; do
  [ "$lib" = "-" ] && L="" || L=$lib
  RSR_B200_LIB=$L timeout 300 python bench.py --config $c --no-cpu --steps 400 --launch $mode 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', '${lib}', '$mode', round(d['ms_per_step']*1e3,3), 'us')"
done; done; done; done
