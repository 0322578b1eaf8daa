"""The reference's DEFAULT mode (adaptive Alg. 1, blocksize 100, tol =
1e-10 ||G||_F; rangefinder.py:68-135) on the device at cfg0/cfg1 shapes:
time per compare() and agreement with the CPU oracle (cfg0 only)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402

for name in ("cfg0", "cfg1"):
    cfg = CONFIGS[name]
    g1, g2 = make_pair(cfg)
    pair = rg.GmpPair.resident(torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda())
    opts = rg.GsvOptions()  # reference defaults
    rep = rg.compare(pair, opts)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 3
    for _ in range(n):
        rep = rg.compare(pair, opts)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    line = f"{name}: adaptive compare() {dt * 1e3:.1f} ms/pair, r={rep.spectrum.r} s={rep.spectrum.s}"
    t0 = time.perf_counter()
    o = orc.run_pipeline(g1, g2, seed=0)
    tc = time.perf_counter() - t0
    line += (f"; CPU oracle {tc * 1e3:.0f} ms, r={o.r} s={o.s}, "
             f"max|alpha - oracle| {np.max(np.abs(rep.spectrum.alphas - o.alphas)):.2e}")
    print(line, flush=True)
