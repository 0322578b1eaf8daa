"""GmpPair rank validation (engine.py:55-61) on the device at cfg1 shapes
(n = 1000): time and compare sigma_max / sigma_min with numpy's SVD."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "cfg1")]
g1, g2 = make_pair(cfg)
t1, t2 = torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pair = rg.GmpPair(t1, t2, check_rank=True)
    torch.cuda.synchronize()
    print(f"device validation: {time.perf_counter() - t0:.3f} s", flush=True)
t0 = time.perf_counter()
s = np.linalg.svd(np.vstack([g1, g2]), compute_uv=False)
print(f"numpy svd: {time.perf_counter() - t0:.3f} s")
print("smax dev %.17e ref %.17e rel %.2e" % (pair.stack_norm2, s[0], abs(pair.stack_norm2 - s[0]) / s[0]))
smin = 1.0 / pair.stack_pinv_norm
print("smin dev %.17e ref %.17e rel %.2e" % (smin, s[-1], abs(smin - s[-1]) / s[-1]))
