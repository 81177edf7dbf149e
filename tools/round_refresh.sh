#!/bin/bash
# Round-end refresh on one GPU: tests, smoke, default bench line, every BASELINE config, the
# ncu launch list of the default bench and one full capture of the scatter kernel.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log
bash tools/bench_all.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 200 --warmup 5 --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launch-list rc=$?"
timeout 300 python tools/prof_multiply.py --iters 3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scatter_kernel -s 2 -c 1 \
    -o gpurun_out/scatter_full -f python tools/prof_multiply.py --iters 3 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
