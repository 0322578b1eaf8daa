"""Generate tests/golden/ref_pipeline.npz by running the REFERENCE's internal
seam engine._run_pipeline + engine.spectrum_from_l_blocks (engine.py:189-261;
called by bench._timed_run, bench.py:74, and cli._cmd_bounds, cli.py:163).

    python tests/golden/make_pipeline_golden.py

Cases: random_pair(40, 30, 20, seed=14) (test_engine.py:189-196) with
method="direct" and the adaptive default (tol 1e-12, seed 15); a
fixed-rank cfg0-structured pair (m=300, p=250, n=80, k=12, q=0). For each:
q1 (None -> absent), l1_block, l2_block, r_tilde, and the spectra of the
three branches (None / "first" / "second")."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import rgsv  # noqa: E402  (the reference)
from rgsv import engine as ref_engine  # noqa: E402
from rgsv.core import gaussian_matrix  # noqa: E402

from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402


def main():
    out = {}
    cases = []
    g1, g2 = gaussian_matrix(40, 20, 14), gaussian_matrix(30, 20, 15)
    cases.append(("direct", g1, g2, rgsv.GsvOptions(method="direct")))
    cases.append(("adaptive", g1, g2, rgsv.GsvOptions(
        extraction=rgsv.ExtractionConfig(tol=1e-12, seed=15))))
    h1, h2 = make_pair(CONFIGS["cfg0"], data_seed=9, m=300, p=250, n=80)
    cases.append(("fixed", h1, h2, rgsv.GsvOptions(extraction=rgsv.ExtractionConfig(
        tol=1e-300, blocksize=12, max_cols=12, trim_tol=0.0, seed=3))))
    for name, a, b, opts in cases:
        pair = rgsv.GmpPair(a, b)
        pl = ref_engine._run_pipeline(pair, opts)
        if pl.q1 is not None:
            out[f"{name}_q1"] = pl.q1
            out[f"{name}_q2"] = pl.q2
        out[f"{name}_l1"] = pl.l1_block
        out[f"{name}_l2"] = pl.l2_block
        out[f"{name}_rt"] = pl.r_tilde
        for br in (None, "first", "second"):
            spec = ref_engine.spectrum_from_l_blocks(pl.l1_block, pl.l2_block, pair.n,
                                                     opts.classify_tol, br)
            tag = br or "merged"
            out[f"{name}_{tag}_alphas"] = spec.alphas
            out[f"{name}_{tag}_betas"] = spec.betas
            out[f"{name}_{tag}_rs"] = np.array([spec.r, spec.s])
    np.savez_compressed(os.path.join(HERE, "ref_pipeline.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
