"""Which neighbour of the multiply launch costs time in the host-buffer loop (16384^2 ternary, int32)."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200 import _native
n = m = 16384
A = (torch.randint(0, 3, (n, m), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, 11)
L = _native.lib(); sp = _native.current_stream_ptr()
vh = torch.randint(-100, 101, (n,), dtype=torch.int32).pin_memory()
dv = torch.empty(n, dtype=torch.int32, device="cuda"); do = torch.empty(m, dtype=torch.int32, device="cuda")
oh = torch.empty(m, dtype=torch.int32).pin_memory()
e = torch.empty(1, device="cuda")
def mult():
    L.rsr_multiply(ctypes.byref(idx.desc), dv.data_ptr(), _native.I32, do.data_ptr(), _native.I32, 1, 0, 0, idx.desc.nblocks, sp)
def t(f, reps=300):
    for _ in range(30): f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6
S = torch.cuda.synchronize
print(f"mult + sync                 {t(lambda: (mult(), S())):7.1f} us")
print(f"H2D + mult + sync           {t(lambda: (dv.copy_(vh, non_blocking=True), mult(), S())):7.1f} us")
print(f"tiny + mult + sync          {t(lambda: (e.add_(1), mult(), S())):7.1f} us")
print(f"H2D + tiny + sync           {t(lambda: (dv.copy_(vh, non_blocking=True), e.add_(1), S())):7.1f} us")
print(f"mult + D2H + sync           {t(lambda: (mult(), oh.copy_(do, non_blocking=True), S())):7.1f} us")
print(f"H2D + mult + D2H + sync     {t(lambda: (dv.copy_(vh, non_blocking=True), mult(), oh.copy_(do, non_blocking=True), S())):7.1f} us")
print(f"launch call only (mult)     {t(lambda: mult()):7.2f} us")
S()
# device time of the kernel launched into an idle GPU
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ds = []
for i in range(200):
    S(); e0.record(); mult(); e1.record(); S()
    if i >= 20: ds.append(e0.elapsed_time(e1) * 1e3)
print(f"event(kernel) isolated       {np.median(ds):7.1f} us")
ds = []
for i in range(200):
    S(); dv.copy_(vh, non_blocking=True); e0.record(); mult(); e1.record(); S()
    if i >= 20: ds.append(e0.elapsed_time(e1) * 1e3)
print(f"event(kernel) after H2D      {np.median(ds):7.1f} us")
ds = []
for i in range(200):
    S(); e0.record(); dv.copy_(vh, non_blocking=True); e1.record(); S()
    if i >= 20: ds.append(e0.elapsed_time(e1) * 1e3)
print(f"event(H2D) isolated          {np.median(ds):7.1f} us")
