"""Host-side cost of one multiply launch vs the wait for it (16384^2 ternary int32)."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200 import _native, kernels as K
n = m = 16384
A = (torch.randint(0, 3, (n, m), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, 11)
L = _native.lib(); sp = _native.current_stream_ptr()
dv = torch.zeros(n, dtype=torch.int32, device="cuda"); do = torch.zeros(m, dtype=torch.int32, device="cuda")
launch, wait, tot = [], [], []
for i in range(400):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.rsr_multiply(ctypes.byref(idx.desc), dv.data_ptr(), _native.I32, do.data_ptr(), _native.I32, 1, 0, 0, idx.desc.nblocks, sp)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if i >= 50:
        launch.append(t1 - t0); wait.append(t2 - t1); tot.append(t2 - t0)
med = lambda x: 1e6 * float(np.median(x))
print(f"launch call {med(launch):.1f} us   wait {med(wait):.1f} us   total {med(tot):.1f} us")
e = torch.empty(1, device="cuda")
def tiny():
    torch.cuda.synchronize(); t0 = time.perf_counter(); e.add_(1); torch.cuda.synchronize(); return time.perf_counter() - t0
print(f"torch tiny op + sync: {med([tiny() for _ in range(300)][50:]):.1f} us")
s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
L.rsr_multiply(ctypes.byref(idx.desc), dv.data_ptr(), _native.I32, do.data_ptr(), _native.I32, 1, 0, 0, idx.desc.nblocks, sp)
t.record(); torch.cuda.synchronize()
print(f"event-timed single launch: {s.elapsed_time(t)*1e3:.1f} us")
