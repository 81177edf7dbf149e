# A/B of the fold-warp count (RSR_B200_FOLD_WARPS; 0 = the built-in choice) on the kernel-only bench value
for c in "$@"; do for fw in ${FWS:-0 1 2 4}; do
  RSR_B200_FOLD_WARPS=$fw timeout 300 python bench.py --config $c --no-cpu --steps 400 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fw=$fw', '$c', round(d['ms_per_step']*1e3,3), 'us')"
done; done
