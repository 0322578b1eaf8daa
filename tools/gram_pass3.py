"""|Q2^T Q2 - I| entering the third CholeskyQR pass on the cfg sketches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402

for name in ("cfg0", "cfg1"):
    cfg = CONFIGS[name]
    g1, _ = make_pair(cfg)
    a = dv.to_device(g1, "g")
    ops = rg.rangefinder._Ops()
    kp, ldn = dv.ceil16(cfg.k), dv.ceil16(cfg.n)
    om = dv.omega_device(cfg.n, cfg.k, [0], ldo=ldn)[0]
    y = torch.zeros((a.rows, kp), dtype=torch.float64, device="cuda")
    ops.gx(dv.vp(a.t), a.ld, dv.vp(om), ldn, dv.vp(y), kp, a.rows, kp, cfg.n)
    for step in range(3):
        gram = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
        ops.gtq(dv.vp(y), kp, dv.vp(y), kp, dv.vp(gram), kp, kp, kp, a.rows)
        e = gram[: cfg.k, : cfg.k].cpu().numpy() - np.eye(cfg.k)
        print(f"{name} pass {step + 1}: max|G - I| = {np.abs(e).max():.2e}  "
              f"|G - I|_F = {np.linalg.norm(e):.2e}")
        linv, _ = ops.chol(gram, cfg.k, kp, a.rows if step == 0 else 0)
        q = torch.zeros_like(y)
        ops.gx(dv.vp(y), kp, dv.vp(linv), kp, dv.vp(q), kp, a.rows, kp, kp)
        y = q
