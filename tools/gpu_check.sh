#!/bin/bash
# One gpurun session: smoke, GPU tests, a short bench, optional ncu capture of the scatter kernel.
#   tools/gpu_check.sh [tests|bench|ncu|all]...
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv,noheader
for what in "${@:-all}"; do
  case $what in
    tests|all)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
      timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
      tail -4 gpurun_out/pytest_gpu.log ;;&
    bench|all)
      timeout 600 python bench.py --cpu-seconds 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
      tail -2 gpurun_out/bench.log ;;&
    ncu|all)
      timeout 300 python tools/prof_multiply.py --iters 3 > gpurun_out/prof_plain.log 2>&1 && \
      timeout 600 ncu --set full --import-source on --clock-control none -k regex:scatter_kernel -s 2 -c 1 \
          -o gpurun_out/scatter_prof -f python tools/prof_multiply.py --iters 3 > gpurun_out/ncu_scatter.log 2>&1
      echo "ncu rc=$?"; cat gpurun_out/prof_plain.log ;;
  esac
done
