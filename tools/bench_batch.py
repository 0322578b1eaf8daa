"""Time rgsv_batch_gsvd on the full cfg3 batch (4096 pairs, resident)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS["cfg3"]
B = int(os.environ.get("B", cfg.batch))
if os.environ.get("DATA", "cfg3") == "gauss":  # plain Gaussian matrices (well conditioned)
    gen = torch.Generator(device="cuda").manual_seed(0)
    g1 = torch.randn((B, cfg.m, cfg.n), generator=gen, device="cuda", dtype=torch.float64)
    g2 = torch.randn((B, cfg.p, cfg.n), generator=gen, device="cuda", dtype=torch.float64)
else:  # the bench's cfg3 data (workloads.py recipe: rank-8 signal + 1e-8 noise)
    import bench
    g1, g2 = bench.device_batch_pairs(cfg, B, 1000)
ALIAS = int(os.environ.get("ALIAS", 0))  # >0: every pair aliases one of ALIAS pairs (L2-resident G)
pairs = [(rg.device.DevMatrix(g1[j % ALIAS if ALIAS else j], cfg.m, cfg.n),
          rg.device.DevMatrix(g2[j % ALIAS if ALIAS else j], cfg.p, cfg.n)) for j in range(B)]
plan = rg.device.small_batch_plan(B, cfg.n, cfg.k)
plan.set_pairs(pairs)
plan.set_seeds([2 * j for j in range(B)])
for _ in range(3):
    plan.launch(cfg.q, 1e-10)
torch.cuda.synchronize()
reps = 10
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(reps):
    plan.launch(cfg.q, 1e-10)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / reps
flops = cfg.flops * B
gbytes = cfg.g_bytes * B / 1e9
print(f"B={B} {ms:.3f} ms/batch  {B / ms * 1e3:.0f} pairs/s  {flops / ms / 1e9:.2f} TF/s "
      f"(alg)  G read once: {gbytes / ms:.0f} GB/s ; 4-pass model {gbytes * 4 / ms:.0f} GB/s")
