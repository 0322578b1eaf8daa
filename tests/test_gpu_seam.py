"""The reference's internal seam on the device: engine._run_pipeline and
engine.spectrum_from_l_blocks (engine.py:189-261), against golden outputs of
the reference itself (tests/golden/make_pipeline_golden.py)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402
from paper_2404_09459_b200 import engine  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_pipeline.npz")


def _cases():
    g1, g2 = orc.gaussian_matrix(40, 20, 14), orc.gaussian_matrix(30, 20, 15)
    h1, h2 = make_pair(CONFIGS["cfg0"], data_seed=9, m=300, p=250, n=80)
    return {
        "direct": (g1, g2, rg.GsvOptions(method="direct")),
        "adaptive": (g1, g2, rg.GsvOptions(extraction=rg.ExtractionConfig(tol=1e-12, seed=15))),
        "fixed": (h1, h2, rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(12, 3, 0))),
    }


@pytest.mark.parametrize("name", ["direct", "adaptive", "fixed"])
def test_run_pipeline_matches_reference(name):
    gold = np.load(GOLD)
    g1, g2, opts = _cases()[name]
    pl = engine._run_pipeline(rg.GmpPair(g1, g2), opts)
    rt = gold[f"{name}_rt"]
    assert pl.r_tilde.shape == rt.shape
    assert np.max(np.abs(pl.r_tilde - rt)) <= 1e-12 * np.abs(rt).max()
    for blk in ("l1", "l2"):
        ref = gold[f"{name}_{blk}"]
        got = getattr(pl, f"{blk}_block")
        assert got.shape == ref.shape
        assert np.max(np.abs(got - ref)) <= 1e-11
    if name == "direct":
        assert pl.q1 is None and pl.q2 is None
    else:
        assert np.max(np.abs(pl.q1 - gold[f"{name}_q1"])) <= 1e-11
        assert np.max(np.abs(pl.q2 - gold[f"{name}_q2"])) <= 1e-11


@pytest.mark.parametrize("name", ["direct", "adaptive", "fixed"])
@pytest.mark.parametrize("branch", [None, "first", "second"])
def test_spectrum_from_l_blocks_matches_reference(name, branch):
    """On the reference's own L blocks: identical r, s; GSVs within 1e-13
    (gesdd vs one-sided Jacobi singular values). Exception, by design of the
    reference (engine.py:198-201): a forced one-sided branch on the
    degenerate fixed-rank blocks (every singular value 1 +- ulp) completes
    sqrt(1 - x^2) from values a rounding away from 1, i.e. sqrt(eps) ~ 1.5e-8
    noise whose classification against 1e-10 depends on the last bit of each
    singular value -- there only the raw side is compared bit-tight and the
    completed side to 4e-8."""
    gold = np.load(GOLD)
    n = gold[f"{name}_rt"].shape[1]
    spec = engine.spectrum_from_l_blocks(gold[f"{name}_l1"], gold[f"{name}_l2"], n, 1e-10,
                                         branch)
    tag = branch or "merged"
    ga, gb = gold[f"{name}_{tag}_alphas"], gold[f"{name}_{tag}_betas"]
    if name == "fixed" and branch is not None:
        raw, comp = (spec.alphas, spec.betas) if branch == "first" else (spec.betas, spec.alphas)
        graw, gcomp = (ga, gb) if branch == "first" else (gb, ga)
        assert np.max(np.abs(raw - graw)) <= 1e-13
        assert np.max(np.abs(comp - gcomp)) <= 4e-8
        return
    assert (spec.r, spec.s) == tuple(int(x) for x in gold[f"{name}_{tag}_rs"])
    assert np.max(np.abs(spec.alphas - ga)) <= 1e-13
    assert np.max(np.abs(spec.betas - gb)) <= 1e-13


def test_seam_composes_like_timed_run():
    """bench._timed_run (bench.py:72-79): _run_pipeline + spectrum_from_l_blocks
    equals compute_gsv."""
    g1, g2, opts = _cases()["adaptive"]
    pair = rg.GmpPair(g1, g2)
    pl = engine._run_pipeline(pair, opts)
    spec = engine.spectrum_from_l_blocks(pl.l1_block, pl.l2_block, pair.n, opts.classify_tol)
    ref = rg.compute_gsv(pair, opts)
    assert (spec.r, spec.s) == (ref.r, ref.s)
    assert np.max(np.abs(spec.alphas - ref.alphas)) <= 1e-12


def test_spectrum_from_l_blocks_rejects_bad_branch():
    with pytest.raises(rg.ValidationError):
        engine.spectrum_from_l_blocks(np.eye(2), np.eye(2), 2, 1e-10, "both")
