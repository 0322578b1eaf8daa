"""GmpPair's default stacked-rank validation at cfg2 size (350000 x 4000):
time and sigma_max / sigma_min, on device-generated cfg2 data."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS["cfg2"]
torch.manual_seed(0)
g1 = torch.randn(cfg.m, cfg.n, dtype=torch.float64, device="cuda")
g2 = torch.randn(cfg.p, cfg.n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
pair = rg.GmpPair(g1, g2)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
smax, smin = pair.stack_norm2, 1.0 / pair.stack_pinv_norm
# Gaussian 350000 x 4000: sigma ~ sqrt(rows) +- sqrt(cols) (Marchenko-Pastur edges)
r, c = cfg.m + cfg.p, cfg.n
print(f"cfg2 GmpPair validation {dt:.1f} s: sigma_max {smax:.6f} (MP edge {r ** .5 + c ** .5:.6f}), "
      f"sigma_min {smin:.6f} (MP edge {r ** .5 - c ** .5:.6f})", flush=True)
