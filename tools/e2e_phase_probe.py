"""Host-buffer session phases for the e2e call (RSR_B200_SESSION_TRACE=1 prints the session's
per-phase medians at exit: stage, enqueue, [D2H wait], wait+convert).
GPU: RSR_B200_SESSION_TRACE=1 python tools/e2e_phase_probe.py [n] [dtype] [copies]"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dt = np.dtype(sys.argv[2]) if len(sys.argv) > 2 else np.dtype(np.float64)
ncopies = int(sys.argv[3]) if len(sys.argv) > 3 else 1
A = (torch.randint(0, 3, (n, n), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
idxs = [rsr.preprocess_ternary(A, rsr.optimal_k_b200(n, n)) for _ in range(ncopies)]
del A
v = np.random.default_rng(0).integers(-100, 101, size=n).astype(dt)
for i in range(50):
    rsr.multiply_ternary(v, idxs[i % ncopies])
ts = []
for i in range(400):
    t = time.perf_counter()
    rsr.multiply_ternary(v, idxs[i % ncopies])
    ts.append(time.perf_counter() - t)
# the device span of one published call: the session graph alone (no host staging / reading)
print(f"n={n} {dt.name} copies={ncopies}: python call median {np.median(ts) * 1e6:.1f} us, p10 {np.percentile(ts, 10) * 1e6:.1f}")
