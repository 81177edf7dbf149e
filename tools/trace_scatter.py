"""Timeline of the scatter kernel from the diagnostic trace build (`make trace`).
GPU: python tools/trace_scatter.py [n]  — prints per-unit stamps (us) of scatter warp 0 / fold warp 0."""
import ctypes, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_06360_b200 import _native
_native.LIB_PATH = os.path.join(ROOT, "paper_2411_06360_b200/lib/trace/librsr_b200_trace.so")
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200 import kernels as K
n = m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
k = rsr.optimal_k_rsrpp(n)
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randint(0, 3, (n, m), device="cuda", dtype=torch.int8, generator=g) - 1).to(torch.int8)
if os.environ.get("TRACE_BINARY"):  # one half: the binary index of the positive entries
    idx = rsr.preprocess(rsr.BinaryMatrix.from_dense((A == 1).to(torch.uint8).cpu().numpy()), k)
else:
    idx = rsr.preprocess_ternary(A, k)
if os.environ.get("TRACE_F32"):  # fp32 activations: the fixed-point (FX) instance
    v = torch.randn(n, device="cuda", generator=g)
    out = torch.empty(m, dtype=torch.float32, device="cuda")
else:
    v = torch.randint(-100, 101, (n,), device="cuda", generator=g).to(torch.int32)
    out = torch.empty(m, dtype=torch.int32, device="cuda")
for _ in range(3):
    K._multiply_device(v, idx, True, None, out)
torch.cuda.synchronize()
if os.environ.get("TRACE_ISOLATED"):  # one launch into an idle GPU (the e2e situation)
    import time
    time.sleep(0.001)
    K._multiply_device(v, idx, True, None, out)
    torch.cuda.synchronize()
buf = np.zeros(148 * 512, np.uint64)
L = _native.lib()
L.rsr_debug_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.rsr_debug_trace_copy(buf.ctypes.data, buf.size) == 0
T = buf.reshape(148, 512).astype(np.float64)
t0 = T[:, 0][T[:, 0] > 0].min()
us = lambda x: (x - t0) / 1e3 if x > 0 else float("nan")
ends = [us(T[c, 7]) for c in range(148)]
print(f"kernel span {np.nanmax(ends):.2f} us; CTA end min/median/max {np.nanmin(ends):.2f}/{np.nanmedian(ends):.2f}/{np.nanmax(ends):.2f}")
starts = sorted(us(T[c, 0]) for c in range(148))
print("CTA start percentiles (us):", [round(starts[i], 2) for i in (0, 37, 74, 111, 147)])
for c in (0, 74, 147):
    print(f"CTA {c}: start {us(T[c,0]):.2f} prefetch {us(T[c,2]):.2f} zeroed {us(T[c,3]):.2f} waited {us(T[c,4]):.2f} "
          f"v_issued {us(T[c,5]):.2f} prologue_end {us(T[c,1]):.2f} end {us(T[c,7]):.2f}")
    for u in range(12):
        r = T[c, 8 + u * 8: 16 + u * 8]
        if r[0] == 0 and r[3] == 0: continue
        print(f"  u{u:2d} scat: top {us(r[0]):6.2f} hfree_ok {us(r[1]):6.2f} reds_done {us(r[2]):6.2f} arrived {us(r[7]):6.2f} tma {us(T[c, 300 + u]):6.2f} | "
              f"fold: start {us(r[3]):6.2f} hfull_ok {us(r[4]):6.2f} read {us(r[5]):6.2f} done {us(T[c, 400 + u]):6.2f}")
