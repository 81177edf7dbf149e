"""Dense 2-bit GEMV launches for ncu: python tools/prof_dense.py"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
n = 16384
A = (torch.randint(0, 3, (n, n), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
D = rsr.DenseTernary(A)
v = torch.randint(-100, 101, (n,), device="cuda").to(torch.int32)
for _ in range(4): D.multiply(v)
torch.cuda.synchronize()
