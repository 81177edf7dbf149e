"""GPU-side work counts: the reference audits its work with instrumented
twins that count the accumulate steps their loops execute (kernels.py:240-320,
test_kernels.py:122-145: n per block for the segmented sums, 2 * 2^w - 2 per block for the RSR++
fold).  The count build of the library (`make count`, csrc/multiply.cu -DRSR_COUNT) has the
scatter kernel count what it actually executes, and this test audits it:

* histogram reductions == halves x rows x blocks exactly (one accumulate per row, half and
  block — the reference's segmented-sum count), and
* fold work (lane adds plus 31 per warp reduction) within 2x the reference's 2 * 2^w - 2 per
  block and half (the GPU fold combines both halves in one histogram and reduces lane bits
  with REDUX, so its count differs from the serial loop's but stays O(2^w) per block).

The count build runs in a subprocess (RSR_B200_LIB selects it), never in the product."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

COUNT_LIB = os.path.join(ROOT, "paper_2411_06360_b200", "lib", "count", "librsr_b200_count.so")

_CHILD = r'''
import ctypes, json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200 import _native
L = _native.lib()
L.rsr_debug_count_copy.argtypes = [ctypes.c_void_p, ctypes.c_int]
out = []
for rows, cols, k, ternary in json.loads(sys.argv[2]):
    rng = np.random.default_rng([rows, cols, k])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8) if ternary else rng.integers(0, 2, size=(rows, cols), dtype=np.int8)
    v = rng.integers(1, 101, size=rows).astype(np.int32) * rng.choice([-1, 1], size=rows).astype(np.int32)  # no zeros
    if ternary:
        idx = rsr.preprocess_ternary(torch.from_numpy(A).cuda(), k)
        mult = rsr.multiply_ternary
    else:
        idx = rsr.preprocess(rsr.BinaryMatrix.from_dense(A.astype(np.uint8)), k)
        mult = rsr.multiply_rsr
    c = np.zeros(4, np.uint64)
    torch.cuda.synchronize()
    L.rsr_debug_count_copy(c.ctypes.data, 1)  # reset
    y = mult(torch.from_numpy(v).cuda(), idx, "rsrpp").cpu().numpy()
    torch.cuda.synchronize()
    L.rsr_debug_count_copy(c.ctypes.data, 1)
    ok = bool(np.array_equal(y.astype(np.int64), v.astype(np.int64) @ A.astype(np.int64)))
    out.append({"red": int(c[0]), "fold": int(c[1]), "redux": int(c[2]), "ok": ok})
print(json.dumps(out))
'''


@pytest.mark.gpu
def test_gpu_work_counts(cuda):
    assert os.path.exists(COUNT_LIB), "build the count library with `make` (target count)"
    cases = [(16384, 600, 11, True), (4096, 1000, 10, True), (1000, 77, 5, True), (2048, 333, 9, False)]
    env = dict(os.environ, RSR_B200_LIB=COUNT_LIB)
    res = subprocess.run([sys.executable, "-c", _CHILD, ROOT, json.dumps(cases)], env=env, capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    got = json.loads(res.stdout.strip().splitlines()[-1])
    for (rows, cols, k, ternary), c in zip(cases, got):
        halves = 2 if ternary else 1
        widths = [min(k, cols - s) for s in range(0, cols, k)]
        assert c["ok"], (rows, cols, k)
        assert c["red"] == halves * rows * len(widths), (rows, cols, k, c)  # exactly the reference's n per block
        ref_fold = halves * sum(2 * (1 << w) - 2 for w in widths)
        gpu_fold = c["fold"] + c["redux"]
        print(f"{rows}x{cols} k={k}: reductions {c['red']}, fold {gpu_fold} vs reference {ref_fold} "
              f"({gpu_fold / ref_fold:.2f}x)")
        assert gpu_fold <= 2 * ref_fold, (rows, cols, k, c)
