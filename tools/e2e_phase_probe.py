"""Host-buffer session phases (RSR_B200_SESSION_TRACE=1 prints medians at exit) for the e2e call."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = (torch.randint(0, 3, (n, n), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, rsr.optimal_k_b200(n, n))
v = np.random.default_rng(0).integers(-100, 101, size=n).astype(np.int32)
for dt in (np.int32, np.float64):
    vv = v.astype(dt)
    for _ in range(50):
        rsr.multiply_ternary(vv, idx)
    ts = []
    for _ in range(300):
        t = time.perf_counter()
        rsr.multiply_ternary(vv, idx)
        ts.append(time.perf_counter() - t)
    print(dt.__name__, "median us", np.median(ts) * 1e6, "p10", np.percentile(ts, 10) * 1e6)
