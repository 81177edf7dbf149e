"""Launch the int32 batched multiply a few times at 16384^2, B=64 (for ncu captures).

    python tools/prof_batched.py [--iters 3] [--batch 64] [--n 16384]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--n", type=int, default=16384)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randint(0, 3, (a.n, a.n), device="cuda", dtype=torch.int8, generator=g) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, rsr.optimal_k_b200(a.n, a.n))
del A
V = torch.randint(-100, 101, (a.batch, a.n), device="cuda", dtype=torch.int32, generator=g)
rsr.multiply_batched(V, idx)  # builds the batch plan
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.iters):
    rsr.multiply_batched(V, idx)
e.record()
torch.cuda.synchronize()
print(f"batched {a.n}^2 B={a.batch}: {s.elapsed_time(e) / a.iters * 1e3:.1f} us per call")
