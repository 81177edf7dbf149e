"""Host-buffer call cost by activation type (4096^2 ternary): int32 vs fp32 vs fp64."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
n = m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A = (torch.randint(0, 3, (n, m), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, rsr.optimal_k_rsrpp(n))
rng = np.random.default_rng(0)
vi = rng.integers(-100, 101, n).astype(np.int32)
vf = rng.standard_normal(n).astype(np.float32)
def t(f, reps=300):
    for _ in range(20): f()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6
print(f"int32 host call   {t(lambda: rsr.multiply_ternary(vi, idx)):7.1f} us")
print(f"fp32 host call    {t(lambda: rsr.multiply_ternary(vf, idx)):7.1f} us")
print(f"fp64 host call    {t(lambda: rsr.multiply_ternary(vf.astype(np.float64), idx)):7.1f} us")
dvf = torch.from_numpy(vf).cuda(); dvi = torch.from_numpy(vi).cuda()
S = torch.cuda.synchronize
print(f"fp32 device+sync  {t(lambda: (rsr.multiply_ternary(dvf, idx), S())):7.1f} us")
print(f"int32 device+sync {t(lambda: (rsr.multiply_ternary(dvi, idx), S())):7.1f} us")
