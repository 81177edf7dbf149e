"""SM clocks while the host-buffer (e2e) loop runs vs while back-to-back kernels run (16384^2)."""
import os, subprocess, sys, threading, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
n = m = 16384
A = (torch.randint(0, 3, (n, m), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, 11)
v = np.random.default_rng(0).integers(-100, 101, n).astype(np.int32)
dv = torch.from_numpy(v).cuda()

def sample(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        out.append(r)
        time.sleep(0.1)

for name, fn in [("e2e numpy", lambda: rsr.multiply_ternary(v, idx)),
                 ("device back-to-back", lambda: rsr.multiply_ternary(dv, idx)),
                 ("device + sync", lambda: (rsr.multiply_ternary(dv, idx), torch.cuda.synchronize()))]:
    for _ in range(200): fn()
    torch.cuda.synchronize()
    stop, out = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, out)); th.start()
    t0 = time.perf_counter(); cnt = 0
    while time.perf_counter() - t0 < 3.0:
        for _ in range(100): fn()
        cnt += 100
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    stop.set(); th.join()
    print(f"{name:22s} {dt / cnt * 1e6:7.1f} us/call  clocks: {out[len(out)//2:len(out)//2+3]}")
