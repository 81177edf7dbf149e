#!/bin/bash
# Final round-2 run on one GPU: GPU tests + smoke, then the full refresh (bench lines of every
# config, launch list, ncu captures; tools/round2_refresh.sh) and the reference arm.
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
rm -rf gpurun_out/r02_bench
bash tools/round2_refresh.sh
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench/reference.json 2>/dev/null; echo "reference rc=$?"
