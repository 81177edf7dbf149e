#!/bin/bash
# A/B of the key-schedule sweeps (preprocess-time knob): kernel time (L2-warm and cold bench) and ncu wavefronts per RED
for sw in 2 4 8; do
  RSR_B200_SCHED_SWEEPS=$sw python tools/prof_multiply.py --config ternary16384 2>&1 | tail -1
  RSR_B200_SCHED_SWEEPS=$sw timeout 300 python bench.py --steps 500 --no-cpu --replays 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sweeps $sw cold us', round(d['ms_per_step']*1e3,2), 'pre', d['notes']['preprocess_s'])"
  RSR_B200_SCHED_SWEEPS=$sw ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_atom.sum -k regex:scatter -s 2 -c 1 python tools/prof_multiply.py --config ternary16384 --iters 3 2>&1 | grep -E "sum" | awk '{print $NF}' | paste -sd' ' | awk '{print "sweeps '$sw' wavefronts/RED", $1/$2}'
done
