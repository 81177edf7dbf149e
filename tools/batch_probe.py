"""Batched multiply timing, both strategies: python tools/batch_probe.py N B"""
import os, sys, subprocess
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
n = int(sys.argv[1]); B = int(sys.argv[2])
k = rsr.optimal_k_rsrpp(n)
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randint(0, 3, (n, n), device="cuda", dtype=torch.int8, generator=g) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, k)
del A
V = torch.randint(-100, 101, (B, n), device="cuda", generator=g).to(torch.int32)
res = {}
for form in ("loop", "gather"):
    os.environ["RSR_B200_BATCH_FORM"] = form
    for _ in range(2): out = rsr.multiply_batched(V, idx)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3): out = rsr.multiply_batched(V, idx)
    e.record(); torch.cuda.synchronize()
    us = s.elapsed_time(e) / 3 * 1e3
    res[form] = out.clone()
    print(f"n={n} B={B} {form}: {us:.0f} us/batch = {B / us * 1e6:,.0f} vectors/s")
print("equal:", bool(torch.equal(res["loop"], res["gather"])))
