"""Launch the batched multiply a few times (for ncu captures): python tools/prof_batched.py [B] [dtype]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dt = getattr(torch, sys.argv[2]) if len(sys.argv) > 2 else torch.int32
n = 16384
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randint(0, 3, (n, n), device="cuda", dtype=torch.int8, generator=g) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, 11)
V = torch.randint(-100, 101, (B, n), device="cuda", generator=g).to(dt)
for _ in range(3):
    rsr.multiply_batched(V, idx)
torch.cuda.synchronize()
print("ok")
