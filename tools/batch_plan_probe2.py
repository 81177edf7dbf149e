import sys, ctypes, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200 import _native, kernels as K
for (rows, cols, k) in [(16384, 600, 11), (8192, 300, 11), (16384, 64, 8)]:
    rng = np.random.default_rng([rows, cols, k])
    A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    idx = rsr.preprocess_ternary(torch.from_numpy(A).cuda(), k)
    bp = K.batch_plan(idx)
    print(rows, cols, k, "plan" if bp else "none", _native.lib().rsr_b200_last_error())
    # expected loads at kb=9
    kb = 9
    nb = (cols + kb - 1) // kb
    worst = 0
    for b in range(nb):
        c0 = b * kb; w = min(kb, cols - c0)
        sub = A[:, c0:c0 + w]
        wts = 1 << np.arange(w - 1, -1, -1)
        kp = ((sub == 1).astype(np.int64) @ wts); kn = ((sub == -1).astype(np.int64) @ wts)
        load = np.bincount(kp, minlength=1 << w) + np.bincount(kn, minlength=1 << w)
        load[0] = 0
        e = int(np.maximum(0, -(-load // 258) - 1).sum())
        worst = max(worst, e)
    print("  host-computed max extra slots:", worst)
