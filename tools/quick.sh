#!/bin/bash
# GPU quick check: gpu tests + smoke + int32/fp32 scatter timings on the BASELINE shapes.
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in ternary16384 llama4096 llama4096x14336 llama14336x4096; do
  for d in int32 float32; do timeout 120 python tools/prof_multiply.py --config $c --dtype $d 2>&1 | tail -1; done
done
timeout 120 python - <<'PY'
import time, torch, numpy as np, sys
sys.path.insert(0, ".")
import paper_2411_06360_b200 as rsr
A = (torch.randint(0, 3, (16384, 16384), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); idx = rsr.preprocess_ternary(A, 11); torch.cuda.synchronize()
    print(f"preprocess 16384^2 k=11: {1e3 * (time.perf_counter() - t):.2f} ms")
PY
timeout 120 python - <<'PY'
import torch, sys
sys.path.insert(0, ".")
import paper_2411_06360_b200 as rsr
n = 16384
A = (torch.randint(0, 3, (n, n), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, 11)
for dt in (torch.int32, torch.float32):
    for B in (64, 128):
        V = torch.randint(-100, 101, (B, n), device="cuda").to(dt)
        for _ in range(3): rsr.multiply_batched(V, idx)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): rsr.multiply_batched(V, idx)
        e.record(); torch.cuda.synchronize()
        us = s.elapsed_time(e) / 10 * 1e3
        print(f"batched {dt} B={B}: {us:.1f} us/batch = {B / us * 1e6:,.0f} vectors/s")
PY
