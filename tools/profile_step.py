"""One warm cfg pipeline step for launch-list profiling, plus a host-side
timing breakdown (Omega generation vs device work).

    python tools/profile_step.py [cfg1] [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402
from paper_2404_09459_b200.engine import run_device_pipeline  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = CONFIGS[name]
g1, g2 = make_pair(cfg)
pair = rg.GmpPair.resident(torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda())
opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))
for _ in range(3):
    run_device_pipeline(pair, opts)
torch.cuda.synchronize()
import numpy as np  # noqa: E402

t0 = time.perf_counter()
for _ in range(20):
    np.random.default_rng(0).standard_normal((cfg.n, cfg.k))
t_om = (time.perf_counter() - t0) / 20
t0 = time.perf_counter()
for i in range(steps):
    run_device_pipeline(pair, opts)
torch.cuda.synchronize()
t_step = (time.perf_counter() - t0) / steps
print(f"{name}: (numpy host omega would cost {t_om*1e3:.3f} ms per matrix); step {t_step*1e3:.3f} ms")
