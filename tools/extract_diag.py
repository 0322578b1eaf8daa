"""Diagnose the low-rank / trim_tol = 0 extraction case of the fuzz sweep:
orthonormality of the basis block by block, device vs oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402

rng = np.random.default_rng(21)
for idx in range(2):
    m = int(rng.integers(2, 3000))
    n = int(rng.integers(2, 400))
    kind = str(rng.choice(["lowrank", "decay", "gauss"]))
    if kind == "lowrank":
        r = int(rng.integers(1, max(2, min(m, n) // 2)))
        g = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    elif kind == "decay":
        r = min(m, n)
        u, _ = np.linalg.qr(rng.standard_normal((m, r)))
        v, _ = np.linalg.qr(rng.standard_normal((n, r)))
        g = (u * 10.0 ** (-6.0 * np.arange(r) / r)) @ v.T
    else:
        g = rng.standard_normal((m, n))
    blocksize = int(rng.choice([1, 3, 8, 17, 50, 100, 128, 200]))
    max_cols = None if rng.random() < 0.5 else int(rng.integers(1, min(m, n) + 1))
    gn = float(np.linalg.norm(g))
    tol = None if rng.random() < 0.3 else gn * 10.0 ** rng.uniform(-6, -1)
    trim_tol = float(rng.choice([1e-12, 1e-8, 0.0]))
    seed = int(rng.integers(0, 1000))
print(kind, m, n, "rank", r, "bs", blocksize, "tol/|G|", tol / gn, "trim", trim_tol)
cfg = rg.ExtractionConfig(tol=tol, blocksize=blocksize, seed=seed, max_cols=max_cols,
                          trim_tol=trim_tol)
ob = orc.extract_basis(g, tol, blocksize, seed, max_cols, trim_tol, 0)
for mode in ("auto", "householder"):
    os.environ["RGSV_ADAPTIVE_QR"] = mode
    res = rg.extract_basis(g, cfg)
    for name, q in (("device/" + mode, res.q), ("oracle", ob.q)):
        k = q.shape[1]
        e = q.T @ q - np.eye(k)
        blocks = [np.abs(e[i:i + blocksize, j:j + blocksize]).max()
                  for i in range(0, k, blocksize) for j in range(0, i + 1, blocksize)]
        print(f"{name:20s} cols={k} orth={np.linalg.norm(e):.2e} worst block entries:",
              " ".join(f"{b:.1e}" for b in blocks))
        print("   col norms of last block:", np.linalg.norm(q[:, -blocksize:], axis=0))
    print("   hist", [f"{h / gn:.2e}" for h in res.residual_history], "oracle",
          [f"{h / gn:.2e}" for h in ob.residual_history])
