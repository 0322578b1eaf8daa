"""Detail of chosen fuzz cases (tools/fuzz_parity.py): basis widths and
residual histories of the adaptive extraction, device vs oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402
from tools.fuzz_parity import make  # noqa: E402

want = {int(x) for x in os.environ.get("IDX", "33,48,52").split(",")}
rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
for i in range(max(want) + 1):
    n = int(rng.integers(3, 260))
    m = int(rng.integers(max(2, n // 3), 1200))
    p = int(rng.integers(max(2, n // 3), 1200))
    if m + p < n:
        m = n
    s = int(rng.integers(1, max(2, min(m, p, n) // 2 + 1)))
    noise = float(rng.choice([1e-3, 1e-6, 1e-9]))
    mode = str(rng.choice(["fixed", "fixed", "direct", "adaptive"]))
    seed = int(rng.integers(0, 1000))
    g1, g2 = make(rng, m, p, n, s, noise)
    if mode == "fixed":
        rng.integers(1, min(m, p, n) + 1)
        rng.integers(0, 3)
    if i not in want:
        continue
    print(f"#{i} m={m} p={p} n={n} s={s} noise={noise:g} mode={mode} seed={seed}")
    for name, g, sd in (("g1", g1, seed), ("g2", g2, seed + 1)):
        res = rg.extract_basis(g, rg.ExtractionConfig(seed=sd))
        ob = orc.extract_basis(g, None, 100, sd, None, 1e-12, 0)
        gn = np.linalg.norm(g)
        true_dev = np.linalg.norm(g - res.q @ (res.q.T @ g)) / gn
        true_orc = np.linalg.norm(g - ob.q @ (ob.q.T @ g)) / gn
        print(f"  {name}: device cols={res.q.shape[1]} widths={res.block_widths} conv={res.converged} "
              f"hist/|G|={[f'{h / gn:.2e}' for h in res.residual_history]} true={true_dev:.2e}")
        print(f"  {name}: oracle cols={ob.q.shape[1]} widths={getattr(ob, 'block_widths', None)} "
              f"conv={getattr(ob, 'converged', None)} "
              f"hist/|G|={[f'{h / gn:.2e}' for h in ob.residual_history]} true={true_orc:.2e}")
