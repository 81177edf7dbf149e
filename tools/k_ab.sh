# Block-width sweep on the kernel-only bench value: tools/k_ab.sh "<k list>" configs...
ks=$1; shift
for c in "$@"; do for k in $ks; do
  timeout 300 python bench.py --config $c --no-cpu --steps 400 --k $k 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', 'k=$k', round(d['ms_per_step']*1e3,3), 'us')"
done; done
