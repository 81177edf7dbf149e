"""Cold timing of the IDP4A dense comparator at 16384^2 (8 rotating copies), for A/B of builds."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
n = 16384
A = (torch.randint(0, 3, (n, n), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
d = rsr.DenseTernary(A)
v = torch.randint(-100, 101, (n,), device="cuda").to(torch.int8)
out = torch.empty(n, dtype=torch.int32, device="cuda")
qs = [d.q] + [d.q.clone() for _ in range(7)]
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
    for i in range(200):
        d.q = qs[i % 8]
        d.multiply_i8(v, out)
torch.cuda.current_stream().wait_stream(s); g.replay(); torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 200 * 1e3)
print(os.environ.get("RSR_B200_LIB", "default"), "dense i8 cold us", round(float(np.median(ts)), 2))
