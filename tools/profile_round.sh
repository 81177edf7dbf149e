#!/bin/bash
# GPU-side: bench + ncu launch list of the same command + one full capture of the scatter kernel.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 200 --warmup 5 --cpu-seconds 2 --no-cpu > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 200 --warmup 5 --no-cpu > gpurun_out/ncu_launches.log 2>&1
echo "launch-list rc=$?"
timeout 300 python tools/prof_multiply.py --iters 3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scatter_kernel -s 2 -c 1 \
    -o gpurun_out/scatter_full -f python tools/prof_multiply.py --iters 3 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
