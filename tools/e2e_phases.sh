# Session (host-buffer) call: phases and device timeline (one GPU).
for n in 4096 16384; do for c in 1 6; do
  RSR_B200_SESSION_TRACE=1 python tools/e2e_phase_probe.py $n float64 $c 2>&1 | grep -v Warn
done; done
RSR_B200_SESSION_TRACE=1 python tools/e2e_phase_probe.py 16384 int32 6 2>&1
RSR_B200_SESSION_TRACE=1 python tools/e2e_phase_probe.py 4096 float32 6 2>&1
(cd tools/microbench && ./session_timeline && COPIES=6 ./session_timeline)
