"""Time the multiply over block ranges [0, nb) to see the per-unit tail cost."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200 import kernels as K
n = m = 16384
k = rsr.optimal_k_rsrpp(n)
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randint(0, 3, (n, m), device="cuda", dtype=torch.int8, generator=g) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, k)
v = torch.randint(-100, 101, (n,), device="cuda", generator=g).to(torch.int32)
out = torch.zeros(m, dtype=torch.int32, device="cuda")
for nb in [int(x) for x in sys.argv[1:]]:
    f = lambda: K._multiply_device(v, idx, True, (0, nb), out)
    for _ in range(3): f()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream(); cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs), torch.cuda.graph(gr, stream=cs):
        for _ in range(50): f()
    torch.cuda.current_stream().wait_stream(cs)
    gr.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(4): gr.replay()
    e.record(); torch.cuda.synchronize()
    us = s.elapsed_time(e) / 200 * 1e3
    print(f"blocks {nb:5d}: {us:6.2f} us  ({us / -(-nb // 148):.2f} us per unit-round)")
