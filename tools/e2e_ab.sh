# A/B of two library builds on the session e2e (tools/e2e_phase_probe.py): tools/e2e_ab.sh <alt.so> "<n dtype copies>"...
alt=$1; shift
for rep in 1 2 3; do for a in "$@"; do for lib in "" "$alt"; do
  echo -n "${lib:-current} $a: "; RSR_B200_LIB=$lib timeout 120 python tools/e2e_phase_probe.py $a 2>&1 | tail -1
done; done; done
