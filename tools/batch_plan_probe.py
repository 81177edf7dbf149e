import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200 import kernels as K
from oracle import c_oracle
for (rows, cols, k, B, vmax) in [(300, 77, 5, 3, 100), (1003, 37, 6, 5, 100), (4096, 333, 10, 70, 100), (16384, 600, 11, 64, 100),
                                 (16384, 601, 11, 64, 30000), (20000, 515, 12, 7, 100), (64, 5, 5, 2, 511)]:
    rng = np.random.default_rng([rows, cols, k, B])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    V = rng.integers(-vmax, vmax + 1, size=(B, rows)).astype(np.int32)
    idx = rsr.preprocess_ternary(torch.from_numpy(A).cuda(), k)
    ref = V.astype(np.int64) @ A.astype(np.int64)
    for variant in ("rsrpp", "rsr"):
        got = rsr.multiply_batched(torch.from_numpy(V).cuda(), idx, variant).cpu().numpy()
        ok = np.array_equal(got.astype(np.int64), ((ref + 2**31) % 2**32) - 2**31)
        print(rows, cols, k, B, vmax, variant, "plan" if idx._bplan else "noplan", "OK" if ok else "MISMATCH", 
              (idx._bplan[0].extra if idx._bplan else None))
        if not ok:
            bad = np.argwhere(got.astype(np.int64) != ref)
            print("  first bad", bad[:5], got[tuple(bad[0])], ref[tuple(bad[0])])
    B2 = (A == 1).astype(np.uint8)
    bidx = rsr.preprocess(rsr.BinaryMatrix.from_dense(B2), k)
    gotb = rsr.multiply_batched(torch.from_numpy(V).cuda(), bidx).cpu().numpy()
    print("  binary", np.array_equal(gotb.astype(np.int64), V.astype(np.int64) @ B2.astype(np.int64)))
# timing 16384^2 B=64
n = 16384
A = (torch.randint(0, 3, (n, n), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, 11)
V = torch.randint(-100, 101, (64, n), device="cuda", dtype=torch.int32)
torch.cuda.synchronize(); t=time.perf_counter(); rsr.multiply_batched(V, idx); torch.cuda.synchronize()
print("first call (plan build) ms", (time.perf_counter()-t)*1e3, "plan", bool(idx._bplan), idx._bplan and idx._bplan[0].extra)
for _ in range(3): rsr.multiply_batched(V, idx)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); s.record()
for _ in range(20): rsr.multiply_batched(V, idx)
e.record(); torch.cuda.synchronize()
print("batched plan 16384^2 B=64: us/batch", s.elapsed_time(e) / 20 * 1e3)
K._PLAN_OFF = True
for _ in range(3): rsr.multiply_batched(V, idx)
torch.cuda.synchronize(); s.record()
for _ in range(20): rsr.multiply_batched(V, idx)
e.record(); torch.cuda.synchronize()
print("old path us/batch", s.elapsed_time(e) / 20 * 1e3)
