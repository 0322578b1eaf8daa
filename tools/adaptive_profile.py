"""Where the adaptive (reference-default) mode spends its time: wraps the
_Ops launch helpers and the small-GSVD stage with synchronized timers."""
import collections
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200 import rangefinder as rf  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402

T = collections.defaultdict(float)
N = collections.Counter()


def wrap(obj, name, label=None):
    fn = getattr(obj, name)

    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        T[label or name] += time.perf_counter() - t0
        N[label or name] += 1
        return out
    setattr(obj, name, w)


for nm in ("gx", "gtq", "chol", "cholqr3", "wide_cholqr3", "householder", "reproject", "sumsq"):
    wrap(rf._Ops, nm)
wrap(rf, "_block_qr")
wrap(rg.device, "small_spectrum")
wrap(rg.device, "device_sumsq")
wrap(rg.device, "omega_block")
cfg = CONFIGS[os.environ.get("CFG", "cfg0")]
g1, g2 = make_pair(cfg)
pair = rg.GmpPair.resident(torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda())
rg.compare(pair, rg.GsvOptions())
T.clear()
N.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
rg.compare(pair, rg.GsvOptions())
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f"total {tot * 1e3:.1f} ms")
for k, v in sorted(T.items(), key=lambda x: -x[1]):
    print(f"{k:16s} {v * 1e3:8.2f} ms  x{N[k]}")
