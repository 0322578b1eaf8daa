"""cfg3: where the host time of compare_batch goes (device-only launch vs
the public call), with a cProfile of the public call."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS["cfg3"]
B = cfg.batch
g1, g2 = bench.device_batch_pairs(cfg, B, 1000)
pairs = [rg.GmpPair.resident(g1[j], g2[j]) for j in range(B)]
base = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))


def step(i):
    return rg.compare_batch(pairs, base, seeds=[2 * (i * B + j) for j in range(B)])


for i in range(3):
    step(i)
torch.cuda.synchronize()
for reps in (5,):
    t0 = time.perf_counter()
    for i in range(reps):
        step(i)
    torch.cuda.synchronize()
    print(f"compare_batch: {(time.perf_counter() - t0) / reps * 1e3:.2f} ms/step")
plan = rg.device.small_batch_plan(B, cfg.n, cfg.k)
t0 = time.perf_counter()
for i in range(5):
    plan.launch(cfg.q, 1e-10)
torch.cuda.synchronize()
print(f"device launch only: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms/step")
pr = cProfile.Profile()
pr.enable()
for i in range(3):
    step(i)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
