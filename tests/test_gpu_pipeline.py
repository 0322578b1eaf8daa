"""End-to-end parity of the B200 pipeline against the reference golden
vectors and the CPU oracle, under the SURVEY.md §0 parity contract:
  (i)  spectrum / comparative quantities: bit-exact vs the reference on the
       fixed-rank configs (the spectrum is data independent there, F2);
  (ii) stage level, identical Omega: captured energy rel <= 1e-13,
       leading-s signal subspace angle <= 1e-12, rows 0..s-1 of B rel
       <= 1e-12, ||Q^T Q - I||_F <= 1e-12 sqrt(k), full span angle <= 1e-6.
"""

import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import rgsv_oracle as orc  # noqa: E402
import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name))


def fixed_opts(k, q=0, seed=0):
    return rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(k, seed, q))


def check_basis(g, res, ob, s_sig, full_tol=1e-6):
    """Stage-level contract for one matrix: device basis vs oracle basis."""
    q = res.q
    k = q.shape[1]
    assert np.linalg.norm(q.T @ q - np.eye(k)) <= 1e-12 * math.sqrt(k)
    assert orc.principal_angles_max(ob.q[:, :s_sig], q[:, :s_sig]) <= 1e-12
    assert orc.principal_angles_max(ob.q, q) <= full_tol
    h_ref = ob.residual_history
    assert abs(res.residual_history[0] - h_ref[0]) <= 1e-14 * h_ref[0]
    e_dev = h_ref[0] ** 2 - res.residual_history[1] ** 2
    b = q.T @ g
    e_ref = orc.sum_sq(ob.q.T @ g)
    assert abs(orc.sum_sq(b) - e_ref) <= 1e-13 * e_ref
    assert abs(e_dev - e_ref) <= 1e-12 * e_ref
    bref = ob.q.T @ g
    assert np.linalg.norm(b[:s_sig] - bref[:s_sig]) <= 1e-12 * np.linalg.norm(bref[:s_sig])


def test_cfg0_q0_spectrum_bit_exact_vs_reference():
    gd = gold("ref_cfg0_q0.npz")
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg)
    pair = rg.GmpPair(g1, g2)
    rep = rg.compare(pair, fixed_opts(cfg.k))
    assert np.array_equal(rep.spectrum.alphas, gd["alphas"])
    assert np.array_equal(rep.spectrum.betas, gd["betas"])
    assert (rep.spectrum.r, rep.spectrum.s) == (int(gd["r"]), int(gd["s"]))
    assert np.array_equal(rep.rho, gd["rho"])
    assert np.max(np.abs(rep.theta - gd["theta"])) <= 1e-15
    assert np.max(np.abs(rep.p1 - gd["p1"])) <= 1e-15
    assert abs(rep.d1 - float(gd["d1"])) <= 1e-14 and abs(rep.d2 - float(gd["d2"])) <= 1e-14


def test_cfg0_q0_stage_parity_vs_reference():
    gd = gold("ref_cfg0_q0.npz")
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg)
    for g, seed, hkey, headkey in ((g1, 0, "hist1", "q1_head"), (g2, 1, "hist2", "q2_head")):
        res = rg.extract_basis(g, rg.ExtractionConfig.fixed_rank(cfg.k, seed, 0))
        ob = orc.fixed_rank_basis(g, cfg.k, 0, seed)
        # the oracle reproduces the reference exactly only on the same BLAS build;
        # across hosts the noise columns (cond ~ 1e9) move at ~1e-8
        assert np.max(np.abs(ob.q[:32, :cfg.s] - gd[headkey][:, :cfg.s])) <= 1e-13
        check_basis(g, res, ob, cfg.s)
        assert abs(res.residual_history[1] - gd[hkey][1]) <= 1e-6 * gd[hkey][0]
        # leading signal columns agree entrywise (same positive-R phase)
        assert np.max(np.abs(res.q[:32, :cfg.s] - gd[headkey][:, :cfg.s])) <= 1e-12


def test_cfg0_q1_vs_oracle():
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg)
    for g, seed in ((g1, 0), (g2, 1)):
        res = rg.extract_basis(g, rg.ExtractionConfig.fixed_rank(cfg.k, seed, cfg.q))
        ob = orc.fixed_rank_basis(g, cfg.k, cfg.q, seed)
        check_basis(g, res, ob, cfg.s)
    spec = rg.compute_gsv(rg.GmpPair(g1, g2), fixed_opts(cfg.k, cfg.q))
    o = orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=0)
    assert np.array_equal(spec.alphas, o.alphas) and (spec.r, spec.s) == (o.r, o.s)


def test_cfg1_full_size_q2():
    cfg = CONFIGS["cfg1"]
    g1, g2 = make_pair(cfg)
    pair = rg.GmpPair(g1, g2)
    run = rg.engine.run_device_pipeline(pair, fixed_opts(cfg.k, cfg.q))
    o = orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=0)
    assert np.array_equal(run.alphas, o.alphas) and (run.r, run.s) == (o.r, o.s)
    for bres, ob in ((run.basis1, o.basis1), (run.basis2, o.basis2)):
        e_ref = orc.sum_sq(ob.b)
        e_dev = bres.residual_history[0] ** 2 - bres.residual_history[1] ** 2
        assert abs(bres.residual_history[0] - ob.residual_history[0]) <= 1e-14 * ob.residual_history[0]
        assert abs(e_dev - e_ref) <= 1e-12 * e_ref
    res = rg.extract_basis(pair.g1, rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))
    check_basis(g1, res, o.basis1, cfg.s)


def test_reference_small_fixed_cases():
    gd = gold("ref_small_fixed.npz")
    for idx in range(3):
        m, p, n, k, seed = (int(x) for x in gd[f"case{idx}"])
        g1 = rg.gaussian_matrix(m, n, 100 + idx)
        g2 = rg.gaussian_matrix(p, n, 200 + idx)
        spec = rg.compute_gsv(rg.GmpPair(g1, g2), fixed_opts(k, 0, seed))
        assert np.array_equal(spec.alphas, gd[f"alphas{idx}"])
        assert [spec.r, spec.s] == list(gd[f"rs{idx}"])
        res = rg.extract_basis(g1, rg.ExtractionConfig.fixed_rank(k, seed, 0))
        e_dev = res.residual_history[0] ** 2 - res.residual_history[1] ** 2
        e_ref = float(gd[f"energy1_{idx}"])
        # Gaussian G has no spectral gap: energy only, at a cond-scaled level
        assert abs(e_dev - e_ref) <= 1e-10 * e_ref


def test_ragged_shapes_vs_oracle():
    rng = np.random.default_rng(3)
    for (m, p, n, k, q) in ((129, 77, 41, 8, 1), (333, 250, 97, 13, 2), (40, 35, 20, 5, 0)):
        u = rng.standard_normal((m, 4)) @ rng.standard_normal((4, n))
        g1 = u + 1e-6 * rng.standard_normal((m, n))
        g2 = rng.standard_normal((p, 4)) @ rng.standard_normal((4, n)) + 1e-6 * rng.standard_normal((p, n))
        res = rg.extract_basis(g1, rg.ExtractionConfig.fixed_rank(k, 0, q))
        ob = orc.fixed_rank_basis(g1, k, q, 0)
        check_basis(g1, res, ob, 4, full_tol=1e-4)
        spec = rg.compute_gsv(rg.GmpPair(g1, g2), fixed_opts(k, q))
        o = orc.run_pipeline(g1, g2, k=k, q=q, seed=0)
        assert np.max(np.abs(spec.alphas - o.alphas)) <= 1e-9
        assert (spec.r, spec.s) == (o.r, o.s)


def test_deterministic_runs():
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg)
    pair = rg.GmpPair(g1, g2)
    a = rg.engine.run_device_pipeline(pair, fixed_opts(cfg.k, cfg.q))
    b = rg.engine.run_device_pipeline(pair, fixed_opts(cfg.k, cfg.q))
    assert a.basis1.residual_history == b.basis1.residual_history
    assert np.array_equal(a.sv1, b.sv1) and np.array_equal(a.theta, b.theta)
    r1 = rg.extract_basis(g1, rg.ExtractionConfig.fixed_rank(cfg.k, 0, 1))
    r2 = rg.extract_basis(g1, rg.ExtractionConfig.fixed_rank(cfg.k, 0, 1))
    assert np.array_equal(r1.q, r2.q)


def test_edge_cases():
    z = np.zeros((7, 5))
    res = rg.extract_basis(z, rg.ExtractionConfig.fixed_rank(3))
    assert res.q.shape == (7, 0) and res.converged and res.iterations == 0
    assert res.residual_history == [0.0]
    bad = np.ones((6, 4))
    bad[2, 1] = np.nan
    with pytest.raises(rg.ValidationError):
        rg.extract_basis(bad, rg.ExtractionConfig.fixed_rank(2))
    with pytest.raises(rg.ValidationError):
        rg.GmpPair(bad, np.ones((3, 4)))
    with pytest.raises(rg.ValidationError):
        rg.extract_basis(np.ones((10, 5)), rg.ExtractionConfig(max_cols=6))
    with pytest.raises(rg.DimensionError):
        rg.GmpPair(np.eye(3), np.eye(4))
    with pytest.raises(rg.RankDeficiencyError):
        rg.GmpPair(rg.gaussian_matrix(2, 6, 1), rg.gaussian_matrix(3, 6, 2))
    with pytest.raises(rg.ValidationError):
        rg.GmpPair(np.eye(2), 1j * np.eye(2))
    with pytest.raises(rg.RecoveryError):  # F2: R-tilde has fewer than n rows
        rg.recover_gsvd(rg.GmpPair(*make_pair(CONFIGS["cfg0"], m=300, p=250)),
                        fixed_opts(30, 1))


def test_analysis_helpers_on_device():
    spec = rg.GsvSpectrum(np.array([0.6]), np.array([0.8]), 0, 1)
    assert rg.angular_distances(spec)[0] == pytest.approx(-0.1418970546041639, abs=1e-15)
    assert rg.relative_significance(spec)[0] == pytest.approx(0.75, abs=1e-15)
    s2 = rg.GsvSpectrum(np.array([1.0, 0.0]), np.array([0.0, 1.0]), 1, 0)
    th = rg.angular_distances(s2)
    assert th[0] == math.pi / 4 and th[1] == -math.pi / 4
    assert rg.relative_significance(s2)[0] == np.inf
    p1, p2 = rg.eigenexpression_fractions(rg.GsvSpectrum(np.array([0.8, 0.6]),
                                                         np.array([0.6, 0.8]), 0, 2))
    assert np.allclose(p1, [0.64, 0.36], atol=1e-15)
    with pytest.raises(rg.DegenerateSpectrumError):
        rg.eigenexpression_fractions(rg.GsvSpectrum(np.array([1.0, 1.0]), np.array([0.0, 0.0]),
                                                    2, 0))
    assert rg.shannon_entropy([1.0, 0.0, 0.0, 0.0]) == 0.0
    assert rg.shannon_entropy([0.5, 0.5, 0.0, 0.0]) == pytest.approx(0.5, abs=1e-15)
    for n in (2, 3, 7, 100):
        assert rg.shannon_entropy(np.full(n, 1.0 / n)) == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(rg.ValidationError):
        rg.shannon_entropy([0.4, 0.4])
    with pytest.raises(rg.ValidationError):
        rg.shannon_entropy([1.0])


def test_rank_check_and_reduced_qr():
    g = rg.gaussian_matrix(50, 20, 4)
    qf = rg.reduced_qr(g)
    assert np.linalg.norm(qf.q @ qf.r - g) <= 1e-12 * np.linalg.norm(g)
    assert np.all(np.diag(qf.r) > 0)
    qr_ref, rr = orc.reduced_qr(g)
    assert np.max(np.abs(qf.q - qr_ref)) <= 1e-12
    u = rg.gaussian_matrix(4, 1, 0)
    with pytest.raises(rg.RankDeficiencyError):
        rg.GmpPair(u @ u.T, u @ u.T, check_rank=True)
    pair = rg.GmpPair(rg.gaussian_matrix(30, 10, 1), rg.gaussian_matrix(25, 10, 2), check_rank=True)
    s = np.linalg.svd(np.vstack([pair.g1.t.cpu().numpy(), pair.g2.t.cpu().numpy()]),
                      compute_uv=False)
    assert abs(pair.stack_norm2 - s[0]) <= 1e-12 * s[0]
    assert abs(pair.stack_pinv_norm - 1 / s[-1]) <= 1e-10 / s[-1]


def test_batch_equals_single():
    cfg = CONFIGS["cfg0"]
    pairs = [rg.GmpPair(*make_pair(cfg, data_seed=d, m=500, p=400)) for d in (1, 2, 3)]
    opts = fixed_opts(cfg.k, cfg.q)
    for _ in range(3):  # eager, capture, replay
        reps = rg.compare_batch(pairs, opts, seeds=[5, 6, 7])
    for pr, rep, seed in zip(pairs, reps, (5, 6, 7)):
        single = rg.compare(pr, fixed_opts(cfg.k, cfg.q, seed))
        assert np.array_equal(rep.spectrum.alphas, single.spectrum.alphas)
        assert np.array_equal(rep.theta, single.theta) and rep.d1 == single.d1
    run = rg.engine.run_device_batch(pairs, opts, seeds=[5, 6, 7])
    ob = orc.fixed_rank_basis(make_pair(cfg, data_seed=2, m=500, p=400)[0], cfg.k, cfg.q, 6)
    e_ref = orc.sum_sq(ob.b)
    h = run[1].basis1.residual_history
    assert abs(h[0] ** 2 - h[1] ** 2 - e_ref) <= 1e-12 * e_ref


def test_rank_check_wide_blocked_cholesky():
    """check_rank=True beyond the one-CTA Cholesky (512 < n <= 1024): the R
    factor comes through the blocked Cholesky; sigma_max / sigma_min agree
    with LAPACK and a rank-deficient stacked pair is rejected like
    engine.py:55-61."""
    rng = np.random.default_rng(3)
    n = 600
    g1 = rng.standard_normal((2000, n))
    g2 = rng.standard_normal((900, n))
    pair = rg.GmpPair(g1, g2, check_rank=True)
    s = np.linalg.svd(np.vstack([g1, g2]), compute_uv=False)
    assert abs(pair.stack_norm2 - s[0]) <= 1e-12 * s[0]
    assert abs(pair.stack_pinv_norm - 1 / s[-1]) <= 1e-10 / s[-1]
    # a stacked pair of rank n - 1 (column n-1 = column 0 + column 1)
    g1[:, -1] = g1[:, 0] + g1[:, 1]
    g2[:, -1] = g2[:, 0] + g2[:, 1]
    with pytest.raises(rg.RankDeficiencyError):
        rg.GmpPair(g1, g2, check_rank=True)


def test_fixed_rank_wide_k():
    """k = 200 (kp = 208 > 128, beyond the fused single-call chain): the pair
    runs the chain as separate launches with every CholeskyQR through the
    blocked Cholesky (stream-ordered scratch), single and batched, and
    matches the oracle."""
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg, data_seed=5, m=3000, p=2500, n=500)
    pair = rg.GmpPair(g1, g2, check_rank=False)
    opts = fixed_opts(200, 1, 4)
    reps = [rg.compare(pair, opts) for _ in range(3)]
    o = orc.run_pipeline(g1, g2, k=200, q=1, seed=4)
    for rep in reps:
        assert np.array_equal(rep.spectrum.alphas, o.alphas)
        assert (rep.spectrum.r, rep.spectrum.s) == (o.r, o.s)
        assert np.array_equal(rep.theta, reps[0].theta)
    pairs = [pair, rg.GmpPair(*make_pair(cfg, data_seed=6, m=3000, p=2500, n=500),
                              check_rank=False)]
    out = rg.compare_batch(pairs, opts, seeds=[4, 9])
    assert np.array_equal(out[0].spectrum.alphas, o.alphas)


def test_extract_basis_wide_fixed_width():
    """extract_basis with a fixed width of 200 (> the fused call's 128):
    same basis contract as the reference (rangefinder.py:68-135)."""
    cfg = CONFIGS["cfg0"]
    g1, _ = make_pair(cfg, data_seed=8, m=2500, p=10, n=400)
    ext = rg.ExtractionConfig.fixed_rank(200, 3, 1)
    res = rg.extract_basis(g1, ext)
    ob = orc.fixed_rank_basis(g1, 200, 1, 3)
    assert res.q.shape == (2500, 200) and res.block_widths == [200]
    assert np.linalg.norm(res.q.T @ res.q - np.eye(200)) <= 1e-12 * np.sqrt(200)
    assert abs(res.residual_history[0] - ob.residual_history[0]) <= 1e-13 * ob.residual_history[0]
    e = res.residual_history[0] ** 2 - res.residual_history[1] ** 2
    eo = orc.sum_sq(ob.b)
    assert abs(e - eo) <= 1e-12 * eo
    s = cfg.s
    qa, _ = np.linalg.qr(res.q[:, :s])
    qb, _ = np.linalg.qr(ob.q[:, :s])
    # sine of the largest principal angle (arccos is blind below ~1e-8)
    assert np.linalg.norm(qb - qa @ (qa.T @ qb), 2) <= 1e-10


def test_host_batch_wide_k():
    """compare_batch on host pairs with k = 200 (> the fused chain) matches
    the oracle."""
    cfg = CONFIGS["cfg0"]
    hosts = [make_pair(cfg, data_seed=d, m=2200, p=2000, n=450) for d in (11, 12)]
    reps = rg.compare_batch(hosts, fixed_opts(200, 1, 0), seeds=[2, 3])
    for (g1, g2), rep, sd in zip(hosts, reps, (2, 3)):
        o = orc.run_pipeline(g1, g2, k=200, q=1, seed=sd)
        assert np.array_equal(rep.spectrum.alphas, o.alphas)
