#!/bin/bash
# Bench-line refresh on one GPU (every BASELINE config, current defaults: independent launches)
# into gpurun_out/r02_bench/, plus the ncu launch list of the default bench.  The per-kernel ncu
# captures come from tools/round2_refresh.sh (kernel bodies unchanged since).
mkdir -p gpurun_out/r02_bench
for c in ternary16384 binary16384 llama4096 llama4096x14336 llama14336x4096 ternary4096f32 ternary16384b64 ternary65536 ternary65536s; do
  timeout 1200 python bench.py --config $c --steps 200 --cpu-seconds 8 > gpurun_out/r02_bench/$c.log 2>&1
  echo "$c rc=$?"; tail -1 gpurun_out/r02_bench/$c.log > gpurun_out/r02_bench/$c.json
done
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench/reference.json 2>/dev/null; echo "reference rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu --replays 2 > gpurun_out/ncu_launches.log 2>&1; echo "launch-list rc=$?"
