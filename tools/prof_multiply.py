"""Launch the single-vector multiply a few times on a BASELINE config (for ncu captures).

    python tools/prof_multiply.py [--config ternary16384] [--iters 5] [--form scatter|gather] [--variant rsrpp|rsr]

Configs follow bench.py (domain, shape, activation dtype); k = indexer.optimal_k_b200 like the bench.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr  # noqa: E402
from paper_2411_06360_b200 import _native, kernels as K  # noqa: E402

CONFIGS = {"ternary16384": ("ternary", 16384, 16384, "int32"), "binary16384": ("binary", 16384, 16384, "int32"),
           "llama4096": ("ternary", 4096, 4096, "int32"), "llama4096x14336": ("ternary", 4096, 14336, "int32"),
           "llama14336x4096": ("ternary", 14336, 4096, "int32"), "ternary65536": ("ternary", 65536, 65536, "int32"),
           "ternary4096f32": ("ternary", 4096, 4096, "float32")}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="ternary16384")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--form", default="scatter")
ap.add_argument("--dtype", default=None)
ap.add_argument("--variant", default="rsrpp")
a = ap.parse_args()
domain, n, m, dtn = CONFIGS[a.config]
dtn = a.dtype or dtn
k = rsr.optimal_k_b200(n, m)
g = torch.Generator(device="cuda").manual_seed(0)
if domain == "ternary":
    A = (torch.randint(0, 3, (n, m), device="cuda", dtype=torch.int8, generator=g) - 1).to(torch.int8)
    idx = rsr.preprocess_ternary(A, k)
else:
    B = np.random.default_rng(0).integers(0, 2, size=(n, m)).astype(np.uint8)
    idx = rsr.preprocess(rsr.BinaryMatrix.from_dense(B), k)
    A = None
del A
dt = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}[dtn]
v = torch.randint(-100, 101, (n,), device="cuda", generator=g).to(dt)
form = {"scatter": _native.FORM_SCATTER, "gather": _native.FORM_GATHER}[a.form]
out = torch.empty(m, dtype=dt, device="cuda")
for _ in range(a.iters):
    K._multiply_device(v, idx, a.variant != "rsr", None, out, form=form)
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
cs.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(cs), torch.cuda.graph(gr, stream=cs):
    for _ in range(20):
        K._multiply_device(v, idx, a.variant != "rsr", None, out, form=form)
torch.cuda.current_stream().wait_stream(cs)
gr.replay()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    gr.replay()
e.record()
torch.cuda.synchronize()
print(f"{a.config} k={k} {a.form} {dtn} {a.variant}: {s.elapsed_time(e) / 100 * 1e3:.1f} us/launch "
      f"(graph of 20 launches, same index: L2-warm)")
