import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2411_06360_b200 as rsr
for (n, m) in [(300, 77), (1000, 513), (16384, 16384)]:
    rng = np.random.default_rng([n, m])
    A = rng.integers(-1, 2, size=(n, m), dtype=np.int8)
    v = rng.integers(-127, 128, size=n).astype(np.int8)
    d = rsr.DenseTernary(torch.from_numpy(A).cuda(), keep_int8=True)
    got = d.multiply_i8(torch.from_numpy(v).cuda()).cpu().numpy()
    ref = v.astype(np.int64) @ A.astype(np.int64)
    print(n, m, "i8 ok", np.array_equal(got, ref))
    if n == 16384:
        dv = torch.from_numpy(v).cuda()
        out = torch.empty(m, dtype=torch.int32, device="cuda")
        for _ in range(3): d.multiply_i8(dv, out)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            for _ in range(50): d.multiply_i8(dv, out)
        torch.cuda.current_stream().wait_stream(s); g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 50 * 1e3
        print("dense i8 GEMV us", us, "GB/s", d.nbytes_i8 / us / 1e3)
        break
        V = torch.from_numpy(rng.integers(-100, 101, size=(64, n)).astype(np.int8)).cuda()
        Y = d.multiply_batched_i8(V)
        print("batched ok", np.array_equal(Y.cpu().numpy(), V.cpu().numpy().astype(np.int64) @ A.astype(np.int64)))
        for _ in range(3): d.multiply_batched_i8(V)
        torch.cuda.synchronize(); e0.record()
        for _ in range(20): d.multiply_batched_i8(V)
        e1.record(); torch.cuda.synchronize()
        print("int8 GEMM B=64 us", e0.elapsed_time(e1) / 20 * 1e3)
