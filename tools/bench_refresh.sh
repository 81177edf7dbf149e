#!/bin/bash
# Bench-only refresh on one GPU: the GPU test suite, every BASELINE config's bench line
# (gpurun_out/r02_bench/<config>.json), the default line and the reference arm.
mkdir -p gpurun_out/r02_bench
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in ternary16384 binary16384 llama4096 llama4096x14336 llama14336x4096 ternary4096f32 ternary16384b64 ternary65536 ternary65536s; do
  timeout 1200 python bench.py --config $c --steps 200 --cpu-seconds 8 > gpurun_out/r02_bench/$c.log 2>&1
  echo "$c rc=$?"; tail -1 gpurun_out/r02_bench/$c.log > gpurun_out/r02_bench/$c.json
done
timeout 300 python bench.py > gpurun_out/default.json 2>gpurun_out/default.err; echo "default rc=$?"; cat gpurun_out/default.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/ref.json
