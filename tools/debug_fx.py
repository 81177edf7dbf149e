import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
from paper_2411_06360_b200 import kernels as K, _native
rows, cols, k = (int(x) for x in sys.argv[1:4])
rng = np.random.default_rng(0)
A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
tidx = rsr.preprocess_ternary(torch.from_numpy(A).cuda(), k)
v = torch.from_numpy(rng.standard_normal(rows).astype(np.float32)).cuda()
out = K._multiply_device(v, tidx, True, form=_native.FORM_SCATTER)
torch.cuda.synchronize()
ref = v.cpu().numpy().astype(np.float64) @ A.astype(np.float64)
print(rows, cols, k, "max err", float(np.abs(out.cpu().numpy() - ref).max()))
