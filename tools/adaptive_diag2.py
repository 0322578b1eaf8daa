"""Adaptive (reference-default) mode at cfg0 shape: dump device vs oracle
block widths, residual histories and spectra."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402

np.set_printoptions(precision=4, linewidth=150)
cfg = CONFIGS[os.environ.get("CFG", "cfg0")]
g1, g2 = make_pair(cfg)
pair = rg.GmpPair(g1, g2)
run = rg.engine.run_device_pipeline(pair, rg.GsvOptions())
o = orc.run_pipeline(g1, g2, seed=0)
for i, (bd, bo) in enumerate(((run.basis1, o.basis1), (run.basis2, o.basis2))):
    print(f"G{i+1}: widths dev {bd.block_widths} ora {bo.block_widths}; "
          f"hist dev {np.array(bd.residual_history)} ora {np.array(bo.residual_history)}")
print("r,s dev", run.r, run.s, "ora", o.r, o.s)
a, b = run.alphas, run.betas
print("dev alphas head", a[:8], "tail", a[-8:])
print("ora alphas head", o.alphas[:8], "tail", o.alphas[-8:])
print("dev betas head", b[:8], "tail", b[-8:])
print("ora betas head", o.betas[:8], "tail", o.betas[-8:])
print("sv1 dev", np.sort(run.sv1)[::-1][:6], np.sort(run.sv1)[:6])
d = np.abs(a - o.alphas)
print("max diff at", int(np.argmax(d)), d.max(), "n diffs > 1e-6:", int((d > 1e-6).sum()))
