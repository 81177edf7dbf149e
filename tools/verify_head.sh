set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/v_smoke.log
timeout 600 python bench.py > gpurun_out/v_default.json 2> gpurun_out/v_default.err; echo "bench rc $?"; cat gpurun_out/v_default.json | head -c 600
timeout 600 python bench.py --impl reference > gpurun_out/v_ref.json 2> gpurun_out/v_ref.err; echo "ref rc $?"; head -c 400 gpurun_out/v_ref.json
