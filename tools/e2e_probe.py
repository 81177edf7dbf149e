"""Where the host-buffer (e2e) call spends its time, 16384^2 ternary int32."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200 import _native, kernels as K
n = m = 16384
A = (torch.randint(0, 3, (n, m), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, 11)
v = np.random.default_rng(0).integers(-100, 101, n).astype(np.int32)
def t(f, reps=300):
    for _ in range(20): f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6
print(f"multiply_ternary(numpy)          {t(lambda: rsr.multiply_ternary(v, idx)):7.1f} us")
plan = K._host_plan(idx, "i32"); out = np.empty(m, np.float64); sp = _native.current_stream_ptr()
print(f"session call (ext, no python)    {t(lambda: plan.call(plan.session, v, out, _native.F64, 1, sp)):7.1f} us")
vh = K._staging.get("v_i32", n, torch.int32, True); dv = K._staging.get("dv_i32", n, torch.int32, False)
oh = K._staging.get("o_f64", m, torch.float64, True); do = K._staging.get("do_f64", m, torch.float64, False)
L = _native.lib(); sp = _native.current_stream_ptr()
def c_call():
    L.rsr_multiply_host(ctypes.byref(idx.desc), vh[2], _native.I32, oh[2], _native.F64, 1, dv[2], do[2], sp)
print(f"rsr_multiply_host (C only)       {t(c_call):7.1f} us")
def kern():
    L.rsr_multiply(ctypes.byref(idx.desc), dv[2], _native.I32, do[2], _native.F64, 1, 0, 0, idx.desc.nblocks, sp)
    torch.cuda.synchronize()
print(f"rsr_multiply + sync (f64 out)    {t(kern):7.1f} us")
def kern32():
    L.rsr_multiply(ctypes.byref(idx.desc), dv[2], _native.I32, do[2], _native.I32, 1, 0, 0, idx.desc.nblocks, sp)
    torch.cuda.synchronize()
print(f"rsr_multiply + sync (i32 out)    {t(kern32):7.1f} us")
def copies():
    dv[0].copy_(vh[0], non_blocking=True); oh[0].copy_(do[0], non_blocking=True); torch.cuda.synchronize()
print(f"H2D 64KB + D2H 128KB + sync      {t(copies):7.1f} us")
print(f"python: stream ptr               {t(lambda: _native.current_stream_ptr(), 3000):7.2f} us")
print(f"python: out copy                 {t(lambda: oh[1].copy(), 3000):7.2f} us")
print(f"python: staging fill             {t(lambda: vh[1].__setitem__(slice(None), v), 3000):7.2f} us")
