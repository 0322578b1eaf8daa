"""Multi-CTA dense kernels (csrc/dense.cu) through the C-ABI, vs numpy/LAPACK.

* rgsv_dense_qr (k_hhqr): blocked Householder QR = the reference's
  core.reduced_qr (core.py:79-96, numpy.linalg.qr + diag(R) >= 0), tall and
  wide, including the stacked form of engine.py:257.
* k_bjacobi through rgsv_svd_values / rgsv_small_gsvd: singular values as
  engine._singular_values (engine.py:228-231) / core.svd (core.py:99-106).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dev  # noqa: E402


def _d(a, ld=None):
    rows, cols = a.shape
    ld = ld or cols + (cols & 1)
    t = torch.zeros((rows, ld), dtype=torch.float64, device="cuda")
    t[:, :cols] = torch.from_numpy(np.ascontiguousarray(a))
    return t


def _st():
    return dev.sp(torch.cuda.current_stream())


def ref_qr(a):
    """core.reduced_qr restated: numpy QR with the diag(R) >= 0 phase fix."""
    q, r = np.linalg.qr(a, mode="reduced")
    d = np.sign(np.diag(r))
    d[d == 0] = 1.0
    return q * d, r * d[:, None]


def dense_qr(a1, a2=None, phase_fix=1):
    L = _native.lib()
    m1, n = a1.shape
    m2 = 0 if a2 is None else a2.shape[0]
    M = m1 + m2
    K = min(M, n)
    A1 = _d(a1)
    A2 = _d(a2) if a2 is not None else None
    Q = torch.full((M, K), np.nan, dtype=torch.float64, device="cuda")
    R = torch.full((K, n), np.nan, dtype=torch.float64, device="cuda")
    nb = int(L.rgsv_dense_qr_workspace_bytes(M, n))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    rc = L.rgsv_dense_qr(dev.vp(A1), A1.stride(0), m1, dev.vp(A2) if A2 is not None else None,
                         A2.stride(0) if A2 is not None else 0, m2, n, dev.vp(Q), K, dev.vp(R), n,
                         phase_fix, dev.vp(ws), nb, _st())
    _native.check(rc, "rgsv_dense_qr")
    return Q.cpu().numpy(), R.cpu().numpy()


QR_SHAPES = [(240, 240), (576, 576), (120, 120), (300, 200), (1000, 64), (60, 200), (33, 17),
             (1408, 40), (700, 700), (5, 1), (1, 9), (130, 4000)]


@pytest.mark.parametrize("m,n", QR_SHAPES)
def test_dense_qr_matches_reduced_qr(m, n):
    rng = np.random.default_rng(m * 1000 + n)
    a = rng.standard_normal((m, n))
    a[:, :1] *= 1e-7  # some spread
    q, r = dense_qr(a)
    qr_, rr_ = ref_qr(a)
    k = min(m, n)
    assert np.linalg.norm(q.T @ q - np.eye(k)) <= 1e-13 * np.sqrt(k)
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.linalg.norm(a)
    assert np.allclose(np.tril(r, -1), 0.0)
    assert np.all(np.diag(r) >= 0)
    # full-rank leading block: the phase-fixed factors are unique
    assert np.max(np.abs(r - rr_)) <= 1e-12 * np.abs(rr_).max()
    assert np.max(np.abs(q - qr_)) <= 1e-9


def test_dense_qr_stacked_two_sources_and_rank_deficient():
    rng = np.random.default_rng(5)
    b1 = rng.standard_normal((150, 400))
    b2 = rng.standard_normal((90, 400))
    b2[7] = b2[3]  # exactly dependent rows of the stack: R_jj -> rounding level
    q, r = dense_qr(b1, b2)
    s = np.vstack([b1, b2])
    assert np.linalg.norm(q.T @ q - np.eye(240)) <= 1e-13 * np.sqrt(240)
    assert np.linalg.norm(q @ r - s) <= 1e-13 * np.linalg.norm(s)
    # a zero column (rank deficiency) keeps tau = 0 like dgeqr2
    z = rng.standard_normal((50, 20))
    z[:, 4] = 0.0
    q2, r2 = dense_qr(z)
    assert abs(r2[4, 4]) == 0.0
    assert np.linalg.norm(q2.T @ q2 - np.eye(20)) <= 1e-13 * np.sqrt(20)
    assert np.linalg.norm(q2 @ r2 - z) <= 1e-13 * np.linalg.norm(z)


def test_dense_qr_rejects_too_many_rows():
    L = _native.lib()
    assert L.rgsv_dense_qr_workspace_bytes(1409, 10) == 0
    rc = L.rgsv_dense_qr(None, 10, 1409, None, 0, 0, 10, None, 10, None, 0, 1, None, 0, None)
    assert rc == 1  # RGSV_ERR_DIMENSION


def svd_values(a, bj_min=None):
    rows, cols = a.shape
    A = _d(a)
    sv = torch.zeros(min(rows, cols), dtype=torch.float64, device="cuda")
    ints = torch.zeros(4, dtype=torch.int32, device="cuda")
    L = _native.lib()
    nb = int(L.rgsv_svd_values_workspace_bytes(rows, cols))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    _native.check(L.rgsv_svd_values(dev.vp(A), A.stride(0), rows, cols, dev.vp(sv),
                                    dev.vp(ints[:2]), dev.vp(ints[2:3]), dev.vp(ws), nb, _st()),
                  "svd")
    assert int(ints[2].item()) == 0, "Jacobi did not converge"
    assert int(ints[0].item()) == min(rows, cols)
    return sv.cpu().numpy()


@pytest.mark.parametrize("rows,cols", [(120, 240), (288, 576), (240, 120), (500, 500), (64, 64),
                                       (33, 1000), (1000, 200), (17, 17), (100, 101)])
def test_blocked_jacobi_values(rows, cols):
    rng = np.random.default_rng(rows + 7 * cols)
    k = min(rows, cols)
    # graded spectrum 1 .. 1e-12 with random singular vectors
    u, _ = np.linalg.qr(rng.standard_normal((rows, k)))
    v, _ = np.linalg.qr(rng.standard_normal((cols, k)))
    s = np.logspace(0, -12, k)
    a = (u * s) @ v.T
    got = svd_values(a)
    ref = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(got - ref)) <= 1e-13 * ref[0]


def test_blocked_jacobi_orthonormal_rows_converge_at_once():
    """The fixed-rank configs feed L blocks with orthonormal rows (F2)."""
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((576, 576)))
    got = svd_values(q[:288])
    assert np.max(np.abs(got - 1.0)) <= 1e-14


@pytest.mark.parametrize("l1,l2,n", [(120, 120, 4000), (288, 288, 8192), (60, 60, 1000),
                                     (150, 150, 200), (200, 90, 250), (100, 40, 141)])
def test_small_gsvd_multicta_vs_lapack(l1, l2, n):
    """rgsv_small_gsvd (k_hhqr + k_bjacobi) = engine.py:257-261 + 228-231."""
    rng = np.random.default_rng(l1 * 3 + l2 + n)
    b1 = rng.standard_normal((l1, n)) * np.logspace(0, -6, n)
    b2 = rng.standard_normal((l2, n)) * np.logspace(-6, 0, n)
    B1, B2 = _d(b1), _d(b2)
    L = _native.lib()
    nb = int(L.rgsv_small_gsvd_workspace_bytes(l1, l2, n))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    r = min(l1 + l2, n)
    sv1 = torch.zeros(max(l1, 1), dtype=torch.float64, device="cuda")
    sv2 = torch.zeros(max(l2, 1), dtype=torch.float64, device="cuda")
    ints = torch.zeros(2, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    _native.check(L.rgsv_small_gsvd(dev.vp(B1), B1.stride(0), l1, dev.vp(B2), B2.stride(0), l2, n,
                                    dev.vp(sv1), dev.vp(sv2), dev.vp(ints), dev.vp(status),
                                    dev.vp(ws), nb, _st()), "small_gsvd")
    assert int(status.item()) == 0
    q = np.linalg.qr(np.vstack([b1, b2]), mode="reduced")[0]
    ref1 = np.linalg.svd(q[:l1], compute_uv=False)
    ref2 = np.linalg.svd(q[l1:], compute_uv=False)
    n1, n2 = int(ints[0].item()), int(ints[1].item())
    assert n1 == min(l1, r) and n2 == min(l2, r)
    assert np.max(np.abs(sv1.cpu().numpy()[:n1] - ref1)) <= 1e-12
    assert np.max(np.abs(sv2.cpu().numpy()[:n2] - ref2)) <= 1e-12


def test_small_gsvd_replay_in_graph():
    """Cooperative launches + memset nodes capture into a CUDA graph and
    replay with changed inputs."""
    rng = np.random.default_rng(11)
    l1 = l2 = 120
    n = 600
    b1 = rng.standard_normal((l1, n))
    b2 = rng.standard_normal((l2, n))
    B1, B2 = _d(b1), _d(b2)
    L = _native.lib()
    nb = int(L.rgsv_small_gsvd_workspace_bytes(l1, l2, n))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    sv1 = torch.zeros(l1, dtype=torch.float64, device="cuda")
    sv2 = torch.zeros(l2, dtype=torch.float64, device="cuda")
    ints = torch.zeros(2, dtype=torch.int32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())

    def run():
        return L.rgsv_small_gsvd(dev.vp(B1), B1.stride(0), l1, dev.vp(B2), B2.stride(0), l2, n,
                                 dev.vp(sv1), dev.vp(sv2), dev.vp(ints), dev.vp(status),
                                 dev.vp(ws), nb, dev.sp(s))

    with torch.cuda.stream(s):
        _native.check(run(), "warm")
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        _native.check(run(), "capture")
    for trial in range(2):
        c1 = rng.standard_normal((l1, n)) * np.logspace(0, -8, n)
        c2 = rng.standard_normal((l2, n))
        B1[:, :n] = torch.from_numpy(c1)
        B2[:, :n] = torch.from_numpy(c2)
        g.replay()
        torch.cuda.synchronize()
        q = np.linalg.qr(np.vstack([c1, c2]), mode="reduced")[0]
        ref1 = np.linalg.svd(q[:l1], compute_uv=False)
        assert np.max(np.abs(sv1.cpu().numpy() - ref1)) <= 1e-12
        assert int(status.item()) == 0
