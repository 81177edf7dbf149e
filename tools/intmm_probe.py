import torch, time
for n in (1024, 4096, 16384):
    a = torch.randint(-100, 101, (64, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-1, 2, (n, n), dtype=torch.int8, device="cuda")
    t = time.time()
    try:
        c = torch._int_mm(a, b); torch.cuda.synchronize()
        print(n, "row-major b ok", time.time() - t, flush=True)
    except Exception as e:
        print(n, "row-major err", e, flush=True)
    bt = b.t().contiguous().t()
    t = time.time()
    c2 = torch._int_mm(a, bt); torch.cuda.synchronize()
    print(n, "col-major b", time.time() - t, flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3): torch._int_mm(a, bt)
    e0.record()
    for _ in range(20): torch._int_mm(a, bt)
    e1.record(); torch.cuda.synchronize()
    print(n, "us", e0.elapsed_time(e1) / 20 * 1e3, flush=True)
