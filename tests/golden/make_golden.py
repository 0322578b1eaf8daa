"""Generate tests/golden/*.npz by running the REFERENCE package itself.

Run here (the container that has /root/reference); the GPU box never reads
/root/reference — it only loads the committed .npz files:

    python tests/golden/make_golden.py

Contents (all from ``rgsv`` 0.1.0 imported from /root/reference/pkg/src):
  ref_cfg0_q0.npz   cfg0 pair (workloads.make_pair), fixed-rank k=30, q=0
                    (ExtractionConfig(tol=1e-300, blocksize=30, max_cols=30,
                    trim_tol=0), as test_bounds.py:71-74): spectrum, r, s,
                    comparative quantities, residual histories, leading rows
                    of Q1/Q2, singular values and energies of B1/B2, raw
                    singular values of the L blocks.
  ref_adaptive.npz  the reference's own oracle-equivalence pairs
                    (test_engine.py:171-179: random_pair seed 7, extraction
                    seed 8, tol 1e-12, real field) in the default adaptive
                    mode: spectra, r, s, theta, block widths.
  ref_small_fixed.npz  small fixed-rank q=0 runs at reference-test shapes.
  oracle_cfg0_q1.npz   the oracle's q=1 restatement on cfg0 (no reference
                    exists for q >= 1: regression vector, parity unpinned).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import rgsv  # noqa: E402  (the reference)
from rgsv import engine as ref_engine  # noqa: E402

from oracle import rgsv_oracle as orc  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402


def unvalidated_pair(g1, g2):
    """GmpPair without the O((m+p)n^2) SVD validation,
    engine only reads g1/g2."""
    pair = object.__new__(rgsv.GmpPair)
    object.__setattr__(pair, "g1", np.asarray(g1, dtype=np.float64))
    object.__setattr__(pair, "g2", np.asarray(g2, dtype=np.float64))
    return pair


def fixed_opts(k, seed=0):
    return rgsv.GsvOptions(
        extraction=rgsv.ExtractionConfig(tol=1e-300, blocksize=k, seed=seed, max_cols=k,
                                          trim_tol=0.0))


def cfg0_q0():
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg)
    pair = rgsv.GmpPair(g1, g2)  # cfg0 is small enough to validate
    opts = fixed_opts(cfg.k)
    pl = ref_engine._run_pipeline(pair, opts)
    spec = ref_engine.spectrum_from_l_blocks(pl.l1_block, pl.l2_block, pair.n, opts.classify_tol)
    rep = rgsv.compare(pair, opts)
    c1 = pl.q1.T @ g1
    c2 = pl.q2.T @ g2
    out = dict(
        alphas=spec.alphas, betas=spec.betas, r=spec.r, s=spec.s,
        rho=rep.rho, theta=rep.theta, p1=rep.p1, p2=rep.p2, d1=rep.d1, d2=rep.d2,
        hist1=np.array(pl.basis1.residual_history), hist2=np.array(pl.basis2.residual_history),
        q1_head=pl.q1[:32].copy(), q2_head=pl.q2[:32].copy(),
        q1_colnorm=np.linalg.norm(pl.q1, axis=0), q2_colnorm=np.linalg.norm(pl.q2, axis=0),
        b1_sv=np.linalg.svd(c1, compute_uv=False), b2_sv=np.linalg.svd(c2, compute_uv=False),
        b1_rows=c1[:20].copy(), b2_rows=c2[:20].copy(),
        energy1=rgsv.core.sum_sq(c1), energy2=rgsv.core.sum_sq(c2),
        l1_sv=np.linalg.svd(pl.l1_block, compute_uv=False),
        l2_sv=np.linalg.svd(pl.l2_block, compute_uv=False),
        stack_smax=pair.stack_norm2, stack_pinv=pair.stack_pinv_norm,
    )
    # the restatement must reproduce the reference bit for bit at q=0
    o = orc.run_pipeline(g1, g2, k=cfg.k, q=0, seed=0)
    assert np.array_equal(o.basis1.q, pl.q1) and np.array_equal(o.basis2.q, pl.q2)
    assert np.array_equal(o.alphas, spec.alphas) and o.basis1.residual_history == pl.basis1.residual_history
    np.savez_compressed(os.path.join(HERE, "ref_cfg0_q0.npz"), **out)


def adaptive():
    shapes = [(60, 45, 30), (25, 70, 40), (35, 30, 50), (40, 30, 20), (30, 40, 20)]
    out = {}
    for idx, (m, p, n) in enumerate(shapes):
        g1 = rgsv.gaussian_matrix(m, n, 7)
        g2 = rgsv.gaussian_matrix(p, n, 8)
        pair = rgsv.GmpPair(g1, g2)
        opts = rgsv.GsvOptions(extraction=rgsv.ExtractionConfig(tol=1e-12, seed=8))
        pl = ref_engine._run_pipeline(pair, opts)
        spec = rgsv.compute_gsv(pair, opts)
        direct = rgsv.compute_gsv(pair, rgsv.GsvOptions(method="direct"))
        rep = rgsv.compare(pair, opts)
        o = orc.run_pipeline(g1, g2, tol=1e-12, seed=8)
        assert np.array_equal(o.alphas, spec.alphas)
        out[f"shape{idx}"] = np.array([m, p, n])
        out[f"alphas{idx}"] = spec.alphas
        out[f"betas{idx}"] = spec.betas
        out[f"direct_alphas{idx}"] = direct.alphas
        out[f"rs{idx}"] = np.array([spec.r, spec.s])
        out[f"theta{idx}"] = rep.theta
        out[f"d{idx}"] = np.array([rep.d1, rep.d2])
        out[f"widths1_{idx}"] = np.array(pl.basis1.block_widths)
        out[f"widths2_{idx}"] = np.array(pl.basis2.block_widths)
        out[f"hist1_{idx}"] = np.array(pl.basis1.residual_history)
    np.savez_compressed(os.path.join(HERE, "ref_adaptive.npz"), **out)


def small_fixed():
    """Fixed-rank q=0 at small shapes, plus the frozen literal."""
    cases = [(300, 250, 64, 16), (500, 400, 100, 24), (129, 77, 40, 8)]
    out = {}
    for idx, (m, p, n, k) in enumerate(cases):
        g1 = rgsv.gaussian_matrix(m, n, 100 + idx)
        g2 = rgsv.gaussian_matrix(p, n, 200 + idx)
        pair = unvalidated_pair(g1, g2)
        opts = fixed_opts(k, seed=idx)
        pl = ref_engine._run_pipeline(pair, opts)
        spec = ref_engine.spectrum_from_l_blocks(pl.l1_block, pl.l2_block, n, opts.classify_tol)
        c1 = pl.q1.T @ g1
        out[f"case{idx}"] = np.array([m, p, n, k, idx])
        out[f"alphas{idx}"] = spec.alphas
        out[f"rs{idx}"] = np.array([spec.r, spec.s])
        out[f"hist1_{idx}"] = np.array(pl.basis1.residual_history)
        out[f"b1_sv{idx}"] = np.linalg.svd(c1, compute_uv=False)
        out[f"energy1_{idx}"] = rgsv.core.sum_sq(c1)
    spec = rgsv.GsvSpectrum(np.array([0.6]), np.array([0.8]), 0, 1)
    out["theta_frozen"] = rgsv.angular_distances(spec)  # test_analysis.py:53-56
    np.savez_compressed(os.path.join(HERE, "ref_small_fixed.npz"), **out)


def oracle_q1():
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg)
    o = orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=0)
    np.savez_compressed(
        os.path.join(HERE, "oracle_cfg0_q1.npz"),
        hist1=np.array(o.basis1.residual_history), hist2=np.array(o.basis2.residual_history),
        b1_sv=np.linalg.svd(o.basis1.b, compute_uv=False),
        b2_sv=np.linalg.svd(o.basis2.b, compute_uv=False),
        alphas=o.alphas, r=o.r, s=o.s)


if __name__ == "__main__":
    cfg0_q0()
    adaptive()
    small_fixed()
    oracle_q1()
    print("golden vectors written to", HERE)
