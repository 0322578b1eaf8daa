"""Per-block orthogonality of the device adaptive range finder (diagnostic)."""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402

base = orc.gaussian_matrix(200, 12, 10)
mix = np.hstack([base + 1e-8 * orc.gaussian_matrix(200, 12, 11) for _ in range(6)])
for mode in ("auto", "householder"):
    os.environ["RGSV_ADAPTIVE_QR"] = mode
    res = rg.extract_basis(mix, rg.ExtractionConfig(tol=1e-300, blocksize=9, seed=12))
    q = res.q
    col = 0
    print(mode, res.block_widths, res.residual_history)
    for w in res.block_widths:
        blk = q[:, col:col + w]
        within = np.linalg.norm(blk.T @ blk - np.eye(w))
        across = np.linalg.norm(q[:, :col].T @ blk) if col else 0.0
        print(f"  block at {col}: within {within:.2e} across {across:.2e}")
        col += w
    o = orc.extract_basis(mix, tol=1e-300, blocksize=9, seed=12)
    print("  oracle widths", o.block_widths, "orth", np.linalg.norm(o.q.T @ o.q - np.eye(o.q.shape[1])))
