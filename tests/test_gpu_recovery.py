"""recover_gsvd on the device (recovery.py) -- mirrors the reference's
TestRecoverGsvd cases (test_engine.py:183-230) plus the F2 rejection of the
fixed-rank BASELINE configs."""

import math

import numpy as np
import pytest

from oracle import rgsv_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg():
    import paper_2404_09459_b200 as rg

    rg._native.require_device()
    return rg


def _random_pair(rg, m, p, n, seed):
    return rg.GmpPair(orc.gaussian_matrix(m, n, seed), orc.gaussian_matrix(p, n, seed + 1))


def _structured_pair(rg, alphas, m, p, seed):
    """G1 = U diag(a) R, G2 = V diag(b) R with prescribed GSVs."""
    alphas = np.asarray(alphas, dtype=np.float64)
    n = alphas.size
    betas = np.sqrt(1.0 - alphas ** 2)
    r_star = orc.gaussian_matrix(n, n, seed)
    u = orc.reduced_qr(orc.gaussian_matrix(m, n, seed + 1))[0]
    v = orc.reduced_qr(orc.gaussian_matrix(p, n, seed + 2))[0]
    return rg.GmpPair(u @ (alphas[:, None] * r_star), v @ (betas[:, None] * r_star))


def _check_factors(pair, fac, g1, g2, tol=1e-8):
    n = g1.shape[1]
    a, b = fac.spectrum.alphas, fac.spectrum.betas
    g1r = fac.u @ (a[:, None] * fac.r_factor)
    g2r = fac.v @ (b[:, None] * fac.r_factor)
    assert np.linalg.norm(g1r - g1) <= tol * max(np.linalg.norm(g1), 1e-30)
    assert np.linalg.norm(g2r - g2) <= tol * max(np.linalg.norm(g2), 1e-30)
    assert np.linalg.norm(fac.u.T @ fac.u - np.eye(n)) <= tol * math.sqrt(n)
    assert np.linalg.norm(fac.v.T @ fac.v - np.eye(n)) <= tol * math.sqrt(n)


@pytest.mark.parametrize("method", ["direct", "randomized"])
@pytest.mark.parametrize("m,p,n", [(40, 30, 20), (30, 40, 20), (300, 260, 120)])
def test_interior_pair_invariants(rg, m, p, n, method):
    g1, g2 = orc.gaussian_matrix(m, n, 14), orc.gaussian_matrix(p, n, 15)
    pair = rg.GmpPair(g1, g2)
    fac = rg.recover_gsvd(pair, rg.GsvOptions(
        method=method, extraction=rg.ExtractionConfig(tol=1e-12, seed=15)))
    _check_factors(pair, fac, g1, g2)


def test_closed_form_proportional(rg):
    g1, g2 = 0.6 * np.eye(2), 0.8 * np.eye(2)
    pair = rg.GmpPair(g1, g2)
    fac = rg.recover_gsvd(pair, rg.GsvOptions(method="direct"))
    _check_factors(pair, fac, g1, g2, tol=1e-10)
    back = fac.u.T @ g1 @ np.linalg.inv(fac.r_factor)
    assert np.allclose(back, 0.6 * np.eye(2), atol=1e-10)


def test_zero_block_completion(rg):
    alphas = np.array([1.0, 1.0, 0.7, 0.4, 0.0])
    pair = _structured_pair(rg, alphas, 30, 25, 16)
    g1, g2 = pair.g1.t.cpu().numpy(), pair.g2.t.cpu().numpy()
    fac = rg.recover_gsvd(pair, rg.GsvOptions(method="direct"))
    assert fac.spectrum.r == 2
    vz = fac.v[:, :2]
    assert np.linalg.norm(vz.T @ vz - np.eye(2)) <= 1e-10
    assert np.linalg.norm(vz.T @ fac.v[:, 2:]) <= 1e-10
    _check_factors(pair, fac, g1, g2)


def test_zero_block_completion_first_branch(rg):
    """l1 <= l2 branch with classified-zero betas (V completion)."""
    alphas = np.array([1.0, 0.9, 0.5, 0.2, 0.1, 0.0])
    pair = _structured_pair(rg, alphas, 20, 40, 26)
    g1, g2 = pair.g1.t.cpu().numpy(), pair.g2.t.cpu().numpy()
    fac = rg.recover_gsvd(pair, rg.GsvOptions(method="direct"))
    assert fac.spectrum.r == 1
    _check_factors(pair, fac, g1, g2)


def test_rejects_wide_shapes(rg):
    pair = _random_pair(rg, 12, 30, 20, 18)
    with pytest.raises(rg.RecoveryError):
        rg.recover_gsvd(pair, rg.GsvOptions(method="direct"))


def test_fixed_rank_degenerate_raises(rg):
    """F2: fixed k with 2k < n leaves fewer than n independent columns."""
    pair = _random_pair(rg, 300, 250, 64, 3)
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(16, 0))
    with pytest.raises(rg.RecoveryError):
        rg.recover_gsvd(pair, opts)


def test_spectrum_matches_compute_gsv(rg):
    pair = _random_pair(rg, 26, 24, 16, 19)
    opts = rg.GsvOptions(method="direct")
    a = rg.recover_gsvd(pair, opts).spectrum
    b = rg.compute_gsv(pair, opts)
    assert np.array_equal(a.alphas, b.alphas) and np.array_equal(a.betas, b.betas)


def test_recovered_spectrum_matches_oracle(rg):
    """GSVs from the recovery equal the restated direct pipeline."""
    g1, g2 = orc.gaussian_matrix(50, 40, 5), orc.gaussian_matrix(45, 40, 6)
    fac = rg.recover_gsvd(rg.GmpPair(g1, g2), rg.GsvOptions(method="direct"))
    qf, _ = orc.reduced_qr(np.vstack([g1, g2]))
    al, be, r, s, *_ = orc.spectrum_from_l_blocks(qf[:50], qf[50:], 40, 1e-10)
    assert np.max(np.abs(fac.spectrum.alphas - al)) <= 1e-12
    assert (fac.spectrum.r, fac.spectrum.s) == (r, s)


@pytest.mark.parametrize("method", ["direct", "randomized"])
def test_wide_pair_blocked_cholesky(rg, method):
    """n = 600 > 512: the stacked QR and every CholeskyQR go through the
    blocked Cholesky (kp > 128); the reference's recovery invariants hold."""
    m, p, n = 900, 700, 600
    g1, g2 = orc.gaussian_matrix(m, n, 21), orc.gaussian_matrix(p, n, 22)
    pair = rg.GmpPair(g1, g2, check_rank=False)
    fac = rg.recover_gsvd(pair, rg.GsvOptions(
        method=method, extraction=rg.ExtractionConfig(tol=1e-12, seed=21)))
    _check_factors(pair, fac, g1, g2)
    qf = rg.reduced_qr(g1)
    assert np.linalg.norm(qf.q @ qf.r - g1) <= 1e-12 * np.linalg.norm(g1)
