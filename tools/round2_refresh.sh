#!/bin/bash
# Round-2 refresh on one GPU: every BASELINE config through bench.py (JSON lines under
# gpurun_out/r02_bench/), the ncu launch list of the default bench, and one `ncu --set full`
# capture of each config's dominant kernel, exported on the box to raw CSV
# (gpurun_out/ncu_<config>_raw.csv; only the headline's .ncu-rep is kept: gpurun_out is capped).
mkdir -p gpurun_out/r02_bench
for c in ternary16384 binary16384 llama4096 llama4096x14336 llama14336x4096 ternary4096f32 ternary16384b64 ternary65536 ternary65536s; do
  timeout 1200 python bench.py --config $c --steps 200 --cpu-seconds 8 > gpurun_out/r02_bench/$c.log 2>&1
  echo "$c rc=$?"; tail -1 gpurun_out/r02_bench/$c.log > gpurun_out/r02_bench/$c.json
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu --replays 2 > gpurun_out/ncu_launches.log 2>&1; echo "launch-list rc=$?"
for c in ternary16384 binary16384 llama4096 llama4096x14336 llama14336x4096 ternary4096f32 ternary65536; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:scatter_kernel -s 2 -c 1 \
      -o gpurun_out/ncu_$c -f python tools/prof_multiply.py --config $c --iters 3 > gpurun_out/ncu_$c.log 2>&1
  echo "ncu $c rc=$?"
  ncu -i gpurun_out/ncu_$c.ncu-rep --page raw --csv > gpurun_out/ncu_${c}_raw.csv 2>/dev/null
  [ "$c" = ternary16384 ] || rm -f gpurun_out/ncu_$c.ncu-rep
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scatter_kernel -s 2 -c 1 \
    -o gpurun_out/ncu_binary16384_rsr -f python tools/prof_multiply.py --config binary16384 --variant rsr --iters 3 > gpurun_out/ncu_binary16384_rsr.log 2>&1
echo "ncu binary rsr rc=$?"
ncu -i gpurun_out/ncu_binary16384_rsr.ncu-rep --page raw --csv > gpurun_out/ncu_binary16384_rsr_raw.csv 2>/dev/null; rm -f gpurun_out/ncu_binary16384_rsr.ncu-rep
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lanes_kernel -s 1 -c 1 \
    -o gpurun_out/ncu_ternary16384b64 -f python tools/prof_batched.py --iters 2 > gpurun_out/ncu_ternary16384b64.log 2>&1
echo "ncu batch rc=$?"
ncu -i gpurun_out/ncu_ternary16384b64.ncu-rep --page raw --csv > gpurun_out/ncu_ternary16384b64_raw.csv 2>/dev/null; rm -f gpurun_out/ncu_ternary16384b64.ncu-rep
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dense_gemv_i8 -s 3 -c 1 \
    -o gpurun_out/ncu_dense16384 -f python tools/dense_probe.py > gpurun_out/ncu_dense.log 2>&1
echo "ncu dense rc=$?"
ncu -i gpurun_out/ncu_dense16384.ncu-rep --page raw --csv > gpurun_out/ncu_dense16384_raw.csv 2>/dev/null; rm -f gpurun_out/ncu_dense16384.ncu-rep
du -sh gpurun_out
