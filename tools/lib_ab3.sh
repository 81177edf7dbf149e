# A/B/C of library builds on the kernel-only bench value: tools/lib_ab3.sh "<lib list>" configs...  ("-" = current)
libs=$1; shift
for rep in 1 2; do for c in "$@"; do for lib in $libs; do
  [ "$lib" = "-" ] && L="" || L=$lib
  RSR_B200_LIB=$L timeout 300 python bench.py --config $c --no-cpu --steps 400 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', '${lib}', round(d['ms_per_step']*1e3,3), 'us')"
done; done; done
