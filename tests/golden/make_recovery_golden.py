"""Generate tests/golden/ref_recovery.npz by running the REFERENCE's own
recover_gsvd (rgsv 0.1.0 from /root/reference/pkg/src, engine.py:294-362).

    python tests/golden/make_recovery_golden.py

Cases (inputs are regenerated in the test from the same seeds):
  interior_{direct,randomized}_{40x30,30x40}  random_pair(m, p, 20, seed=14)
        with ExtractionConfig(tol=1e-12, seed=15) (test_engine.py:189-196)
  zero_block   structured_pair([1, 1, .7, .4, 0], 30, 25, seed=16), direct
        (test_engine.py:205-214)
  cfg0_adaptive  a reduced-row cfg0 pair (workloads.make_pair(cfg0,
        data_seed=3, m=400, p=300, n=120)) in the reference's default
        adaptive mode with blocksize 70 and tol 1.0 (far above the 1e-8 noise
        floor, so Alg. 1 stops after one block on both sides: l1 = l2 = 70,
        l1 + l2 = 140 > n: interior GSVs, no rounding-level stop decision -- DESIGN.md §2)
For each: U, V, R, alphas, betas, r, s.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import rgsv  # noqa: E402  (the reference)
from rgsv.core import gaussian_matrix, reduced_qr  # noqa: E402

from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402


def random_pair(m, p, n, seed):
    return gaussian_matrix(m, n, seed), gaussian_matrix(p, n, seed + 1)


def structured(alphas, m, p, seed):
    alphas = np.asarray(alphas, dtype=np.float64)
    n = alphas.size
    betas = np.sqrt(1.0 - alphas ** 2)
    r_star = gaussian_matrix(n, n, seed)
    u = reduced_qr(gaussian_matrix(m, n, seed + 1)).q
    v = reduced_qr(gaussian_matrix(p, n, seed + 2)).q
    return u @ (alphas[:, None] * r_star), v @ (betas[:, None] * r_star)


def main():
    out = {}

    def run(name, g1, g2, opts):
        fac = rgsv.recover_gsvd(rgsv.GmpPair(g1, g2), opts)
        out[f"{name}_u"] = fac.u
        out[f"{name}_v"] = fac.v
        out[f"{name}_r"] = fac.r_factor
        out[f"{name}_alphas"] = fac.spectrum.alphas
        out[f"{name}_betas"] = fac.spectrum.betas
        out[f"{name}_rs"] = np.array([fac.spectrum.r, fac.spectrum.s])

    for method in ("direct", "randomized"):
        for m, p in ((40, 30), (30, 40)):
            g1, g2 = random_pair(m, p, 20, 14)
            run(f"interior_{method}_{m}x{p}", g1, g2, rgsv.GsvOptions(
                method=method, extraction=rgsv.ExtractionConfig(tol=1e-12, seed=15)))
    g1, g2 = structured([1.0, 1.0, 0.7, 0.4, 0.0], 30, 25, 16)
    run("zero_block", g1, g2, rgsv.GsvOptions(method="direct"))
    g1, g2 = make_pair(CONFIGS["cfg0"], data_seed=3, m=400, p=300, n=120)
    run("cfg0_adaptive", g1, g2, rgsv.GsvOptions(extraction=rgsv.ExtractionConfig(
        tol=1.0, blocksize=70, seed=0)))
    np.savez_compressed(os.path.join(HERE, "ref_recovery.npz"), **out)
    print("wrote", sorted(out)[:4], "...", len(out), "arrays")


if __name__ == "__main__":
    main()
