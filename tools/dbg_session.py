import os, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2411_06360_b200 as rsr
from oracle import c_oracle
n, m, k = int(sys.argv[1]), int(sys.argv[2]), 11
rng = np.random.default_rng(0)
A = rng.integers(-1, 2, size=(n, m), dtype=np.int8)
idx = rsr.preprocess_ternary(torch.from_numpy(A).cuda(), k)
v = rng.integers(-100, 101, size=n).astype(np.int32)
ref = c_oracle.naive_ternary(v.astype(np.float64), A)
for i in range(8):
    t = time.perf_counter()
    try:
        got = rsr.multiply_ternary(v, idx)
    except Exception as e:
        print("call", i, "failed after", time.perf_counter() - t, "s:", e, flush=True); break
    print("call", i, "ok" if np.array_equal(got, ref) else "WRONG", round((time.perf_counter() - t) * 1e6, 1), "us", flush=True)
