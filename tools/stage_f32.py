"""Stage times of the cfg4 (fp32, chunked) pipeline, synchronized per stage."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS["cfg4"]
frac = float(os.environ.get("FRAC", "1"))
m, p = int(cfg.m * frac), int(cfg.p * frac)
g1 = torch.randn((m, cfg.n), device="cuda", dtype=torch.float32)
g2 = torch.randn((p, cfg.n), device="cuda", dtype=torch.float32)
d1 = dv.DevMatrix(g1, m, cfg.n)
d2 = dv.DevMatrix(g2, p, cfg.n)


def t(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    print(f"{label:28s} {(time.perf_counter() - t0) * 1e3:9.1f} ms", flush=True)
    return out


for rep in range(2):
    print("rep", rep)
    _, b1, _ = t("chain G1 (chunked)", lambda: rg.rangefinder.chunked_chain(d1, cfg.k, cfg.q, 0))
    _, b2, _ = t("chain G2 (chunked)", lambda: rg.rangefinder.chunked_chain(d2, cfg.k, cfg.q, 1))
    t("small GSVD + comparative", lambda: dv.small_spectrum(b1, cfg.k, b2, cfg.k, cfg.n, 1e-10))
    ops = rg.rangefinder._Ops()
    y = torch.randn((m, dv.ceil16(cfg.k)), device="cuda", dtype=torch.float64)
    t("cholqr3 on Y (m x kp)", lambda: ops.cholqr3(y, m, cfg.k, dv.ceil16(cfg.k)))
    t("sumsq f32 (chunked)", lambda: dv.device_sumsq(d1))
