"""e2e of non-integer float64 vectors through the host session: the fixed-point route
(max / min nonzero |v| <= 2^21) vs the fp64 gather kernel (a vector with a wider range).
GPU: python tools/e2e_float_probe.py"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200.kernels import classify_host_vector
for n in (4096, 16384):
    A = (torch.randint(0, 3, (n, n), device="cuda", dtype=torch.int8) - 1).to(torch.int8)
    idx = rsr.preprocess_ternary(A, rsr.optimal_k_b200(n, n))
    v = np.random.default_rng(0).standard_normal(n)
    vw = v.copy()
    vw[7] = 1e-9  # dynamic range beyond 2^21: the fp64 gather kernel
    for vec in (v, vw):
        for _ in range(20):
            rsr.multiply_ternary(vec, idx)
        ts = []
        for _ in range(200):
            t = time.perf_counter()
            rsr.multiply_ternary(vec, idx)
            ts.append(time.perf_counter() - t)
        print(n, classify_host_vector(vec)[0], "fp64 float e2e median us", round(np.median(ts) * 1e6, 1))
