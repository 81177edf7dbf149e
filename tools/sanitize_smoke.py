"""Small runs of the round-2 paths for compute-sanitizer (memcheck / racecheck / synccheck):
host sessions (pull + streamed tags, every staging class), the batch plan kernel with staged
codes, the fused all-gather epilogue with virtual ranks.
GPU: python tools/sanitize_smoke.py (compute-sanitizer is closed on this pool)"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200 import dist as D
from oracle import c_oracle

rng = np.random.default_rng(1)
for rows, cols, k in ((3000, 777, 8), (16384, 301, 11)):
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    idx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
    for it in range(3):
        v = rng.integers(-100, 101, size=rows)
        ref = c_oracle.naive_ternary(v.astype(np.float64), A)
        assert np.array_equal(rsr.multiply_ternary(v.astype(np.float64), idx), ref)
        assert np.array_equal(rsr.multiply_ternary(v.astype(np.int32), idx, "rsr"), ref)
        vf = rng.standard_normal(rows)
        np.testing.assert_allclose(rsr.multiply_ternary(vf, idx), c_oracle.naive_ternary(vf, A), rtol=1e-9, atol=1e-9)
        rsr.multiply_ternary(vf.astype(np.float32), idx)
        big = v.astype(np.int64) * (1 << 30)
        rsr.multiply_ternary(big, idx)
    V = torch.from_numpy(rng.integers(-100, 101, size=(5, rows)).astype(np.int32)).cuda()
    out = rsr.multiply_batched(V, idx)
    for b in range(5):
        assert np.array_equal(out[b].cpu().numpy().astype(np.float64), c_oracle.naive_ternary(V[b].cpu().numpy().astype(np.float64), A))
# fused all-gather, 3 virtual ranks
rows, cols, k, world = 2048, 300, 9, 3
A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
idxs = [D.preprocess_ternary_shard(A, k, world, r) for r in range(world)]
pad = max(D.slice_lengths(cols, k, world))
g = [torch.zeros(2, world * pad, dtype=torch.int32, device="cuda") for _ in range(world)]
sg = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(world)]
dn = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(world)]
f = [D.FusedAllGather(idxs[r], cols, world, r, [(x[0].data_ptr(), x[1].data_ptr()) for x in g],
                      [s.data_ptr() for s in sg], g[r], dn[r]) for r in range(world)]
for call in range(3):
    v = rng.integers(-100, 101, size=rows).astype(np.int32)
    dv = torch.from_numpy(v).cuda()
    for x in f:
        x.launch(dv)
    ref = c_oracle.naive_ternary(v.astype(np.float64), A)
    for x in f:
        assert np.array_equal(x.wait().cpu().numpy().astype(np.float64), ref)
torch.cuda.synchronize()
print("sanitize smoke ok")
