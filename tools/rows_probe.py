import os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200 import kernels as K
for n in (int(x) for x in sys.argv[1:]):
    m = 16384
    A = (torch.randint(0, 3, (n, m), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
    idx = rsr.preprocess_ternary(A, 11)
    v = torch.randint(-100, 101, (n,), device="cuda").to(torch.int32)
    out = torch.empty(m, dtype=torch.int32, device="cuda")
    f = lambda: K._multiply_device(v, idx, True, None, out)
    for _ in range(3): f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(20): f()
    torch.cuda.current_stream().wait_stream(s); g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): g.replay()
    b.record(); torch.cuda.synchronize()
    print(f"rows {n}: {a.elapsed_time(b) / 100 * 1e3:.1f} us")
