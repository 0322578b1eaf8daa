"""GmpPair rank validation and core.reduced_qr on the device beyond the
round-1 limits (reference engine.py:40-90, core.py:79-96).

* validation: stacked R factor (Householder <= 1408 rows, CholeskyQR3 above,
  n <= 4096) + blocked Jacobi; sigma_max / sigma_min vs LAPACK.
* reduced_qr: tall and wide, Householder / CholeskyQR3 / rank-deficient
  fallback, against numpy.linalg.qr with the reference's phase fix.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402


def _check_qr(a, tol_q=1e-10):
    qf = rg.reduced_qr(a)
    q_ref, r_ref = orc.reduced_qr(a)
    k = min(a.shape)
    assert qf.q.shape == q_ref.shape and qf.r.shape == r_ref.shape
    assert np.linalg.norm(qf.q.T @ qf.q - np.eye(k)) <= 1e-13 * np.sqrt(k) * 10
    assert np.linalg.norm(qf.q @ qf.r - a) <= 1e-13 * np.linalg.norm(a) * 10
    assert np.all(np.diag(qf.r) >= 0)
    assert np.array_equal(np.tril(qf.r, -1), np.zeros_like(np.tril(qf.r, -1)))
    assert np.max(np.abs(qf.r - r_ref)) <= 1e-11 * np.abs(r_ref).max()
    assert np.max(np.abs(qf.q - q_ref)) <= tol_q
    return qf


@pytest.mark.parametrize("rows,cols", [(30, 80), (600, 1500), (1408, 1408), (3000, 50),
                                       (20000, 300), (1500, 1600)])
def test_reduced_qr_tall_and_wide(rows, cols):
    rng = np.random.default_rng(rows + cols)
    _check_qr(rng.standard_normal((rows, cols)))


def test_reduced_qr_rank_deficient_tall_beyond_householder_rows():
    """rows > 1408 with an exactly dependent column: CholeskyQR breaks down
    and the one-CTA Householder kernel takes over (the reference permits
    rank deficiency, core.py:82-84)."""
    rng = np.random.default_rng(7)
    a = rng.standard_normal((3000, 40))
    a[:, 5] = a[:, 2]
    qf = rg.reduced_qr(a)
    assert np.linalg.norm(qf.q.T @ qf.q - np.eye(40)) <= 1e-12
    assert np.linalg.norm(qf.q @ qf.r - a) <= 1e-12 * np.linalg.norm(a)
    assert abs(qf.r[5, 5]) <= 1e-12 * np.abs(np.diag(qf.r)).max()


@pytest.mark.parametrize("m,p,n", [(20000, 16000, 1000), (4000, 3000, 1500), (700, 600, 400)])
def test_default_rank_check_large_n(m, p, n):
    """The default GmpPair now validates cfg1-sized pairs and n > 1024 (the
    reference always validates, engine.py:55-61)."""
    rng = np.random.default_rng(n)
    g1 = rng.standard_normal((m, n))
    g2 = rng.standard_normal((p, n)) * np.logspace(0, -4, n)
    pair = rg.GmpPair(g1, g2)
    s = np.linalg.svd(np.vstack([g1, g2]), compute_uv=False)
    assert abs(pair.stack_norm2 - s[0]) <= 1e-12 * s[0]
    assert abs(pair.stack_pinv_norm - 1 / s[-1]) <= 1e-9 / s[-1]


def test_rank_deficient_pair_rejected_by_default():
    rng = np.random.default_rng(2)
    n = 1200
    g1 = rng.standard_normal((3000, n))
    g2 = rng.standard_normal((2000, n))
    g1[:, 7] = 2.0 * g1[:, 3]
    g2[:, 7] = 2.0 * g2[:, 3]
    with pytest.raises(rg.RankDeficiencyError):
        rg.GmpPair(g1, g2)


def test_lazy_stack_norms_when_check_skipped():
    rng = np.random.default_rng(4)
    g1 = rng.standard_normal((900, 300))
    g2 = rng.standard_normal((800, 300))
    pair = rg.GmpPair(g1, g2, check_rank=False)
    s = np.linalg.svd(np.vstack([g1, g2]), compute_uv=False)
    assert abs(pair.stack_norm2 - s[0]) <= 1e-12 * s[0]
    assert abs(pair.stack_pinv_norm - 1 / s[-1]) <= 1e-10 / s[-1]


def test_rank_check_beyond_limit_is_explicit():
    """n > 4096 with more than 1408 stacked rows: an explicit DimensionError
    instead of a silently skipped check."""
    g = torch.zeros((2100, 4200), dtype=torch.float64, device="cuda")
    g.normal_()
    with pytest.raises(rg.DimensionError):
        rg.GmpPair(g, g.clone())
    pair = rg.GmpPair(g, g.clone(), check_rank=False)
    with pytest.raises(rg.DimensionError):
        _ = pair.stack_norm2


@pytest.mark.parametrize("rows,cols", [(2100, 2200), (2300, 150)])
def test_svd_with_vectors_blocked(rows, cols):
    """core.svd (core.py:99-106) beyond the one-CTA Jacobi's 2048 vectors:
    blocked Jacobi with accumulated rotations; values vs LAPACK,
    reconstruction and orthonormal factors."""
    rng = np.random.default_rng(rows)
    a = rng.standard_normal((rows, cols))
    f = rg.svd(a)
    ref = np.linalg.svd(a, compute_uv=False)
    k = min(rows, cols)
    assert np.max(np.abs(f.s - ref)) <= 1e-12 * ref[0]
    assert np.linalg.norm((f.u * f.s) @ f.v.T - a) <= 1e-12 * np.linalg.norm(a)
    assert np.linalg.norm(f.u.T @ f.u - np.eye(k)) <= 1e-11 * np.sqrt(k)
    assert np.linalg.norm(f.v.T @ f.v - np.eye(k)) <= 1e-11 * np.sqrt(k)


@pytest.mark.parametrize("rows,n,smin", [(3000, 300, 3e-12), (6000, 1100, 2e-11)])
def test_ill_conditioned_full_rank_stack_is_accepted(rows, n, smin):
    """A stack with sigma_min / sigma_max above the reference's 1e-12 rank
    threshold (engine.py:57-61) is a valid pair, however ill conditioned: the
    CholeskyQR3 route used beyond 1408 stacked rows breaks down there in its
    unshifted second pass and is retried with two shifted passes (found by
    tools/fuzz_parity.py: such pairs were rejected as rank deficient)."""
    rng = np.random.default_rng(rows + n)
    u, _ = np.linalg.qr(rng.standard_normal((rows, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    sig = np.logspace(0.0, np.log10(smin), n)
    s = (u * sig) @ v.T
    cut = rows * 3 // 5
    pair = rg.GmpPair(s[:cut], s[cut:])  # must not raise
    sv = np.linalg.svd(s, compute_uv=False)
    assert abs(pair.stack_norm2 - sv[0]) <= 1e-12 * sv[0]
    assert abs(1.0 / pair.stack_pinv_norm - sv[-1]) <= 0.05 * sv[-1]
    # ... and the direct method factors it (stacked QR beyond the Householder
    # rows: two shifted + two plain CholeskyQR passes), at the conditioning-
    # scaled distance from the oracle's LAPACK result
    spec = rg.compute_gsv(pair, rg.GsvOptions(method="direct"))
    o = orc.run_pipeline(s[:cut], s[cut:], direct=True)
    tol = 200.0 * 2.220446049250313e-16 * sv[0] / sv[-1]
    assert (spec.r, spec.s) == (o.r, o.s)
    assert np.max(np.abs(spec.alphas - o.alphas)) <= tol
    pl = rg.engine._run_pipeline(pair, rg.GsvOptions(method="direct"))
    q = np.vstack([pl.l1_block, pl.l2_block])
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 1e-12 * np.sqrt(n)
    # the same matrix pushed below the threshold is still rejected
    sig2 = sig.copy()
    sig2[-1] = 1e-14
    s2 = (u * sig2) @ v.T
    with pytest.raises(rg.RankDeficiencyError):
        rg.GmpPair(s2[:cut], s2[cut:])
