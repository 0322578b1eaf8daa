"""Direct method and the adaptive range finder (Alg. 1) on the device.

Pinned against the reference's own outputs (tests/golden/ref_adaptive.npz,
made by tests/golden/make_golden.py from rgsv 0.1.0) and against the oracle's
restatement of rangefinder.py:68-135; the property tests mirror the
reference's test_engine.py / test_rangefinder.py cases.
"""

import math

import numpy as np
import pytest

from oracle import rgsv_oracle as orc

pytestmark = pytest.mark.gpu

GOLDEN = "tests/golden/ref_adaptive.npz"


@pytest.fixture(scope="module")
def rg():
    import paper_2404_09459_b200 as rg

    rg._native.require_device()
    return rg


def _pair(m, p, n, seed):
    return orc.gaussian_matrix(m, n, seed), orc.gaussian_matrix(p, n, seed + 1000)


def _adaptive(rg, tol=1e-12, seed=8, **kw):
    return rg.GsvOptions(extraction=rg.ExtractionConfig(tol=tol, seed=seed, **kw))


# ------------------------------------------------------------ golden vectors
def test_adaptive_and_direct_match_reference_golden(rg):
    gd = np.load(GOLDEN)
    for idx in range(5):
        m, p, n = (int(x) for x in gd[f"shape{idx}"])
        g1 = orc.gaussian_matrix(m, n, 7)
        g2 = orc.gaussian_matrix(p, n, 8)
        pair = rg.GmpPair(g1, g2)
        run = rg.engine.run_device_pipeline(pair, _adaptive(rg))
        assert np.max(np.abs(run.alphas - gd[f"alphas{idx}"])) <= 1e-12, idx
        assert np.max(np.abs(run.betas - gd[f"betas{idx}"])) <= 1e-12, idx
        assert [run.r, run.s] == list(gd[f"rs{idx}"]), idx
        assert np.max(np.abs(run.theta - gd[f"theta{idx}"])) <= 1e-11, idx
        assert run.basis1.block_widths == list(gd[f"widths1_{idx}"]), idx
        assert run.basis2.block_widths == list(gd[f"widths2_{idx}"]), idx
        h = gd[f"hist1_{idx}"]
        assert math.isclose(run.basis1.residual_history[0], h[0], rel_tol=1e-14)
        # after full capture the cumulative residual sqrt(max(|G|^2 - sum, 0))
        # (rangefinder.py:126-127) sits at the rounding floor, sqrt(a few ulp
        # of |G|^2) ~ 1e-7 |G|: both sides must be at that floor
        assert abs(run.basis1.residual_history[1] - h[1]) <= 2e-7 * h[0]
        d1, d2 = gd[f"d{idx}"]
        assert abs(run.d1 - d1) <= 1e-12 and abs(run.d2 - d2) <= 1e-12
        direct = rg.compute_gsv(pair, rg.GsvOptions(method="direct"))
        assert np.max(np.abs(direct.alphas - gd[f"direct_alphas{idx}"])) <= 1e-12, idx


# ------------------------------------------------- test_engine.py mirrors
def test_fully_separated_pair(rg):
    pair = rg.GmpPair(np.diag([1.0, 0.0]), np.diag([0.0, 1.0]))
    spec = rg.compute_gsv(pair, rg.GsvOptions(method="direct"))
    assert np.array_equal(spec.alphas, [1.0, 0.0])
    assert np.array_equal(spec.betas, [0.0, 1.0])
    assert (spec.r, spec.s) == (1, 0)


def test_proportional_identities(rg):
    pair = rg.GmpPair(0.6 * np.eye(2), 0.8 * np.eye(2))
    for method in ("direct", "randomized"):
        spec = rg.compute_gsv(pair, rg.GsvOptions(method=method))
        assert np.allclose(spec.alphas, 0.6, atol=1e-12)
        assert np.allclose(spec.betas, 0.8, atol=1e-12)
        assert (spec.r, spec.s) == (0, 2)


@pytest.mark.parametrize("m,p,n", [(60, 45, 30), (25, 70, 40), (35, 30, 50)])
def test_direct_vs_randomized(rg, m, p, n):
    g1, g2 = _pair(m, p, n, 7)
    pair = rg.GmpPair(g1, g2)
    direct = rg.compute_gsv(pair, rg.GsvOptions(method="direct"))
    rand = rg.compute_gsv(pair, _adaptive(rg))
    gap = max(np.max(np.abs(direct.alphas - rand.alphas)), np.max(np.abs(direct.betas - rand.betas)))
    assert gap <= 1e-8


def test_pythagorean_and_scale_covariance(rg):
    for seed in range(3):
        g1, g2 = _pair(20 + seed, 25, 15, seed)
        spec = rg.compute_gsv(rg.GmpPair(g1, g2), rg.GsvOptions(method="direct"))
        assert np.max(np.abs(spec.alphas ** 2 + spec.betas ** 2 - 1)) <= 1e-12
    g1, g2 = _pair(30, 28, 20, 9)
    base = rg.compute_gsv(rg.GmpPair(g1, g2), rg.GsvOptions(method="direct"))
    for c in (1e-3, 1e3):
        spec = rg.compute_gsv(rg.GmpPair(c * g1, c * g2), rg.GsvOptions(method="direct"))
        assert np.max(np.abs(spec.alphas - base.alphas)) <= 1e-10


def test_zero_first_matrix(rg):
    pair = rg.GmpPair(np.zeros((4, 3)), orc.gaussian_matrix(5, 3, 11))
    for opts in (rg.GsvOptions(method="direct"), rg.GsvOptions()):
        spec = rg.compute_gsv(pair, opts)
        assert np.array_equal(spec.alphas, np.zeros(3))
        assert np.array_equal(spec.betas, np.ones(3))
        assert (spec.r, spec.s) == (0, 0)


def test_wide_first_matrix(rg):
    g1, g2 = _pair(12, 30, 20, 12)
    pair = rg.GmpPair(g1, g2)
    direct = rg.compute_gsv(pair, rg.GsvOptions(method="direct"))
    assert np.all(direct.alphas[12:] == 0.0)
    rand = rg.compute_gsv(pair, _adaptive(rg, seed=13))
    assert np.max(np.abs(direct.alphas - rand.alphas)) <= 1e-8


def test_direct_matches_oracle_pipeline(rg):
    """Direct method against the restated stacked-QR + SVD (engine.py:246-261)."""
    g1, g2 = _pair(140, 90, 64, 21)
    spec = rg.compute_gsv(rg.GmpPair(g1, g2), rg.GsvOptions(method="direct"))
    qf, _ = orc.reduced_qr(np.vstack([g1, g2]))
    al, be, r, s, *_ = orc.spectrum_from_l_blocks(qf[:140], qf[140:], 64, 1e-10)
    assert np.max(np.abs(spec.alphas - al)) <= 1e-12
    assert (spec.r, spec.s) == (r, s)


# --------------------------------------------- test_rangefinder.py mirrors
def _basis(rg, g, **kw):
    return rg.extract_basis(g, rg.ExtractionConfig(**kw))


def test_zero_matrix_terminates_before_sampling(rg):
    res = _basis(rg, np.zeros((7, 5)), tol=1e-8)
    assert res.q.shape == (7, 0) and res.converged and res.iterations == 0
    assert res.residual_history == [0.0]


def test_rank_one_gives_single_column(rg):
    rng = np.random.default_rng(0)
    u = rng.standard_normal((100, 1))
    v = rng.standard_normal((50, 1))
    g = (u / np.linalg.norm(u)) @ (v / np.linalg.norm(v)).T
    res = _basis(rg, g, tol=1e-10, blocksize=10, seed=1, trim_tol=1e-12)
    assert res.q.shape[1] == 1
    assert rg.residual_norm(g, res.q) <= 1e-10


@pytest.mark.parametrize("shape,bs,seed,iters", [((120, 120), 25, 3, 5), ((40, 23), 10, 5, 3)])
def test_full_saturation_and_uneven_final_block(rg, shape, bs, seed, iters):
    g = orc.gaussian_matrix(*shape, seed - 1)
    res = _basis(rg, g, tol=1e-300, blocksize=bs, seed=seed)
    assert res.iterations == iters
    assert res.q.shape[1] <= shape[1]
    assert rg.residual_norm(g, res.q) <= 1e-10 * np.linalg.norm(g)


def test_cumulative_residual_matches_explicit(rg):
    g = orc.gaussian_matrix(80, 40, 8)
    u, _, vt = np.linalg.svd(g, full_matrices=False)
    g = u @ np.diag(np.geomspace(1, 1e-6, 40)) @ vt
    res = _basis(rg, g, tol=1e-300, blocksize=7, seed=9)
    assert len(res.residual_history) == res.iterations + 1
    assert np.all(np.diff(res.residual_history) <= 1e-10)
    nrm = np.linalg.norm(g)
    col = 0
    for i, width in enumerate(res.block_widths, start=1):
        col += width
        explicit = rg.residual_norm(g, res.q[:, :col])
        assert abs(res.residual_history[i] - explicit) <= 1e-8 * nrm


def test_orthogonality_drift_bounded(rg):
    base = orc.gaussian_matrix(200, 12, 10)
    mix = np.hstack([base + 1e-8 * orc.gaussian_matrix(200, 12, 11) for _ in range(6)])
    res = _basis(rg, mix, tol=1e-300, blocksize=9, seed=12)
    l = res.q.shape[1]
    assert np.linalg.norm(res.q.T @ res.q - np.eye(l)) <= 1e-11 * math.sqrt(l)


def test_trim_disabled_keeps_all_sampled_columns(rg):
    rng = np.random.default_rng(13)
    g = rng.standard_normal((50, 1)) @ rng.standard_normal((30, 1)).T
    res = _basis(rg, g, tol=1e-300, blocksize=10, seed=14, trim_tol=0.0)
    assert res.q.shape[1] == 30
    assert np.linalg.norm(res.q.T @ res.q - np.eye(30)) <= 1e-11 * math.sqrt(30)


def test_max_cols_mid_loop_and_wide_saturation(rg):
    g = orc.gaussian_matrix(60, 40, 17)
    res = _basis(rg, g, tol=1e-300, blocksize=4, seed=18, max_cols=10, trim_tol=0.0)
    assert res.q.shape[1] == 10 and res.block_widths == [4, 4, 2]
    w = orc.gaussian_matrix(20, 60, 20)
    res = _basis(rg, w, tol=1e-300, blocksize=12, seed=21)
    assert res.q.shape[1] <= 20
    assert rg.residual_norm(w, res.q) <= 1e-10 * np.linalg.norm(w)


def test_same_seed_same_basis_bitwise(rg):
    g = orc.gaussian_matrix(30, 18, 22)
    cfg = rg.ExtractionConfig(tol=1e-6, blocksize=6, seed=23)
    r1, r2 = rg.extract_basis(g, cfg), rg.extract_basis(g, cfg)
    assert np.array_equal(r1.q, r2.q) and r1.residual_history == r2.residual_history


@pytest.mark.parametrize("m,n,bs,decay", [(300, 120, 50, 1e-5), (500, 250, 100, 1e-6),
                                          (90, 45, 5, 1e-4), (64, 200, 16, 1e-3)])
def test_adaptive_matches_oracle_restatement(rg, m, n, bs, decay):
    """Same block widths, iterations and convergence as the oracle's Alg. 1
    restatement; residual histories and the spanned subspace agree to
    roundoff. The spectrum has a clean gap (decay, then exact zeros) so the
    trim test (|R_jj| >= 1e-12 |G|) and the stop test are decided far from
    the rounding floor on both sides."""
    g = orc.gaussian_matrix(m, n, 31)
    u, _, vt = np.linalg.svd(g, full_matrices=False)
    r = min(m, n)
    sv = np.geomspace(1, decay, r)
    sv[int(0.7 * r):] = 0.0  # exact rank deficiency -> trimming
    g = (u[:, :r] * sv) @ vt[:r]
    tol = 1e-5 * np.linalg.norm(g)  # well above the ~1e-7 |G| rounding floor
    o = orc.extract_basis(g, tol=tol, blocksize=bs, seed=5)
    d = _basis(rg, g, tol=tol, blocksize=bs, seed=5)
    assert d.block_widths == o.block_widths and d.iterations == o.iterations
    assert d.converged == o.converged
    # compare residual ENERGIES (|G|^2 - captured): near full capture the
    # norm itself is sqrt of rounding noise, the energy is not
    nrm = o.residual_history[0]
    e_d = np.array(d.residual_history) ** 2
    e_o = np.array(o.residual_history) ** 2
    assert np.max(np.abs(e_d - e_o)) <= 1e-13 * nrm ** 2
    # the same subspace: Q_o^T Q_d is orthogonal
    c = o.q.T @ d.q
    sv_c = np.linalg.svd(c, compute_uv=False)
    assert np.max(np.abs(sv_c - 1.0)) <= 1e-8


def test_adaptive_power_iters_matches_oracle(rg):
    g = orc.gaussian_matrix(400, 150, 41)
    o = orc.extract_basis(g, tol=1e-300, blocksize=40, seed=3, max_cols=80, power_iters=1)
    d = _basis(rg, g, tol=1e-300, blocksize=40, seed=3, max_cols=80, power_iters=1)
    assert d.block_widths == o.block_widths
    nrm = o.residual_history[0]
    e_d = np.array(d.residual_history) ** 2
    e_o = np.array(o.residual_history) ** 2
    assert np.max(np.abs(e_d - e_o)) <= 1e-12 * nrm ** 2


def test_sketch_wider_than_rank_keeps_columns_like_reference(rg):
    """Exactly low-rank input, fixed width above the rank, trim_tol = 0: the
    reference's Householder QR keeps all `width` columns (rangefinder.py:
    119-124); the fused CholeskyQR path breaks down there and must fall back
    to the general loop instead of raising (found by the randomized sweep).
    The captured energy and the spectrum agree with the oracle."""
    rng = np.random.default_rng(5)
    g1 = rng.standard_normal((900, 6)) @ rng.standard_normal((6, 80))
    g2 = rng.standard_normal((700, 6)) @ rng.standard_normal((6, 80)) \
        + 1e-3 * rng.standard_normal((700, 80))
    cfg = rg.ExtractionConfig.fixed_rank(20, 3, 0)
    res = rg.extract_basis(g1, cfg)
    ob = orc.fixed_rank_basis(g1, 20, 0, 3)
    assert res.q.shape == ob.q.shape == (900, 20) and res.block_widths == [20]
    assert abs(res.residual_history[0] - ob.residual_history[0]) <= 1e-13 * ob.residual_history[0]
    # the 6 real directions span range(g1): nothing of g1 is left
    assert np.linalg.norm(g1 - res.q @ (res.q.T @ g1)) <= 1e-7 * np.linalg.norm(g1)
    assert np.linalg.norm(res.q[:, :6].T @ res.q[:, :6] - np.eye(6)) <= 1e-12
    spec = rg.compute_gsv(rg.GmpPair(g1, g2, check_rank=False),
                          rg.GsvOptions(extraction=cfg))
    o = orc.run_pipeline(g1, g2, k=20, q=0, seed=3)
    assert (spec.r, spec.s) == (o.r, o.s)
