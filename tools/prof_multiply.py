"""Launch the multiply kernel a few times on a BASELINE config (for ncu captures).

    python tools/prof_multiply.py [--config ternary16384] [--iters 5] [--form scatter|gather] [--dtype int32|float32]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr  # noqa: E402
from paper_2411_06360_b200 import _native, kernels as K  # noqa: E402

SHAPES = {"ternary16384": (16384, 16384), "llama4096": (4096, 4096), "llama4096x14336": (4096, 14336),
          "llama14336x4096": (14336, 4096), "ternary65536": (65536, 65536)}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="ternary16384")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--form", default="scatter")
ap.add_argument("--dtype", default="int32")
ap.add_argument("--variant", default="rsrpp")
a = ap.parse_args()
n, m = SHAPES[a.config]
k = rsr.optimal_k_rsrpp(n)
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randint(0, 3, (n, m), device="cuda", dtype=torch.int8, generator=g) - 1).to(torch.int8)
idx = rsr.preprocess_ternary(A, k)
del A
dt = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64}[a.dtype]
v = torch.randint(-100, 101, (n,), device="cuda", generator=g).to(dt)
form = {"scatter": _native.FORM_SCATTER, "gather": _native.FORM_GATHER}[a.form]
out = torch.empty(m, dtype=dt, device="cuda")
for _ in range(a.iters):
    K._multiply_device(v, idx, a.variant != "rsr", None, out, form=form)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
cs.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
    for _ in range(20):
        K._multiply_device(v, idx, a.variant != "rsr", None, out, form=form)
torch.cuda.current_stream().wait_stream(cs)
g.replay()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    g.replay()
e.record()
torch.cuda.synchronize()
print(f"{a.config} {a.form} {a.dtype} {a.variant}: {s.elapsed_time(e) / 100 * 1e3:.1f} us/launch "
      f"(graph of 20 launches, same index: L2-warm)")
