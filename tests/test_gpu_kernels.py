"""Kernel-level parity on the B200 through the C-ABI (each vs numpy fp64)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dev  # noqa: E402


def _even(x):
    return x + (x & 1)


def _dev(a, ld=None):
    rows, cols = a.shape
    ld = ld or _even(cols)
    t = torch.zeros((rows, ld), dtype=torch.float64, device="cuda")
    t[:, :cols] = torch.from_numpy(a)
    return t


def _scratch(nbytes=256 << 20):
    return torch.empty(nbytes, dtype=torch.uint8, device="cuda")


def _st():
    return dev.sp(torch.cuda.current_stream())


def relerr(x, y):
    return np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)


GX_SHAPES = [(2000, 32, 200), (20000, 64, 1000), (129, 16, 77), (5, 64, 40), (300, 128, 64),
             (1000, 256, 100), (64, 64, 1000), (4000, 16, 64), (16000, 64, 1000),
             (5003, 288, 288), (777, 192, 50), (130, 384, 96)]  # 96-wide tiles (N % 96 == 0)


@pytest.mark.parametrize("M,N,K", GX_SHAPES)
def test_gemm_gx(M, N, K):
    rng = np.random.default_rng(M * 7 + N + K)
    a = rng.standard_normal((M, K))
    bt = rng.standard_normal((N, K))
    A, Bt = _dev(a), _dev(bt)
    C = torch.zeros((M, _even(N)), dtype=torch.float64, device="cuda")
    S = _scratch()
    rc = _native.lib().rgsv_gemm_gx(dev.vp(A), A.stride(0), dev.vp(Bt), Bt.stride(0), dev.vp(C),
                                    C.stride(0), M, N, K, dev.vp(S), S.numel(), _st())
    _native.check(rc, "gx")
    got = C[:, :N].cpu().numpy()
    assert relerr(got, a @ bt.T) <= 1e-14


GTQ_SHAPES = [(20000, 64, 1000), (2000, 32, 200), (77, 16, 130), (4000, 16, 64), (64, 64, 1000),
              (1000, 128, 64), (20000, 64, 64), (3000, 48, 64), (200, 256, 96)]


@pytest.mark.parametrize("K,M,N", GTQ_SHAPES)
def test_gemm_gtq(K, M, N):
    rng = np.random.default_rng(K + 3 * M + N)
    a = rng.standard_normal((K, M))
    b = rng.standard_normal((K, N))
    A, B = _dev(a), _dev(b)
    C = torch.zeros((M, _even(N)), dtype=torch.float64, device="cuda")
    S = _scratch()
    rc = _native.lib().rgsv_gemm_gtq(dev.vp(A), A.stride(0), dev.vp(B), B.stride(0), dev.vp(C),
                                     C.stride(0), M, N, K, dev.vp(S), S.numel(), _st())
    _native.check(rc, "gtq")
    got = C[:, :N].cpu().numpy()
    assert relerr(got, a.T @ b) <= 1e-14


def test_gemm_deterministic():
    rng = np.random.default_rng(5)
    a = rng.standard_normal((20000, 1000))
    q = rng.standard_normal((20000, 64))
    A, Q = _dev(a), _dev(q)
    S = _scratch()
    outs = []
    for _ in range(2):
        C = torch.zeros((64, 1008), dtype=torch.float64, device="cuda")
        _native.check(_native.lib().rgsv_gemm_gtq(dev.vp(Q), 64, dev.vp(A), A.stride(0),
                                                  dev.vp(C), 1008, 64, 1000, 20000, dev.vp(S),
                                                  S.numel(), _st()), "gtq")
        outs.append(C.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("k", [1, 5, 16, 60, 64, 120, 129, 240, 288, 300, 576, 700])
def test_chol_inv(k):
    kp = (k + 15) // 16 * 16
    rng = np.random.default_rng(k)
    x = rng.standard_normal((3 * k + 5, k))
    a = x.T @ x
    G = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
    G[:k, :k] = torch.from_numpy(a)
    linv = torch.zeros(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
    rinv = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
    rd = torch.zeros(kp, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = _native.lib().rgsv_chol_inv(dev.vp(G), k, kp, 0, dev.vp(linv), dev.vp(rinv), dev.vp(rd),
                                     dev.vp(status), _st())
    _native.check(rc, "chol")
    assert int(status.item()) == 0
    Li = linv[: kp * kp].view(kp, kp).cpu().numpy()
    L = np.linalg.cholesky(a)
    assert relerr(Li[:k, :k], np.linalg.inv(L)) <= 1e-12
    assert np.array_equal(Li[k:, k:], np.eye(kp - k))
    assert np.array_equal(rinv.cpu().numpy(), Li.T)
    assert relerr(rd[:k].cpu().numpy(), np.diag(L)) <= 1e-13


@pytest.mark.parametrize("k", [16, 288])
def test_chol_breakdown_flag(k):
    kp = k
    G = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")  # singular
    linv = torch.zeros(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    _native.check(_native.lib().rgsv_chol_inv(dev.vp(G), k, kp, 0, dev.vp(linv), None, None,
                                              dev.vp(status), _st()), "chol")
    assert int(status.item()) & _native.ST_CHOL


@pytest.mark.parametrize("rows,cols", [(30, 60), (60, 120), (45, 20), (1, 7), (128, 128)])
def test_svd_values(rows, cols):
    rng = np.random.default_rng(rows * cols)
    a = rng.standard_normal((rows, cols))
    a[:, 0] *= 1e-6  # spread the spectrum
    A = _dev(a)
    sv = torch.zeros(min(rows, cols), dtype=torch.float64, device="cuda")
    ints = torch.zeros(4, dtype=torch.int32, device="cuda")
    nb = int(_native.lib().rgsv_svd_values_workspace_bytes(rows, cols))
    ws = _scratch(nb)
    _native.check(_native.lib().rgsv_svd_values(dev.vp(A), A.stride(0), rows, cols, dev.vp(sv),
                                                dev.vp(ints[:2]), dev.vp(ints[2:3]), dev.vp(ws),
                                                nb, _st()), "svd")
    ref = np.linalg.svd(a, compute_uv=False)
    got = sv.cpu().numpy()
    assert int(ints[0].item()) == min(rows, cols)
    assert int(ints[2].item()) == 0
    assert np.max(np.abs(got - ref)) <= 1e-13 * ref[0]
    # relative accuracy of the smallest values (one-sided Jacobi property)
    assert np.max(np.abs(got - ref) / ref) <= 1e-10


def test_comparative_kernel_vs_oracle():
    from oracle import rgsv_oracle as orc

    rng = np.random.default_rng(11)
    n, l1, l2 = 50, 30, 30
    q, _ = np.linalg.qr(rng.standard_normal((l1 + l2, n)))  # 60 x 50 orthonormal columns
    o_al, o_be, r, s, v1, v2 = orc.spectrum_from_l_blocks(q[:l1], q[l1:], n)
    out = torch.zeros(6 * n + 4, dtype=torch.float64, device="cuda")
    ints = torch.zeros(8, dtype=torch.int32, device="cuda")
    ints[1], ints[2] = v1.size, v2.size
    s1 = torch.from_numpy(v1).cuda()
    s2 = torch.from_numpy(v2).cuda()
    rc = _native.lib().rgsv_comparative(
        dev.vp(s1), dev.vp(ints[1:3]), dev.vp(s2), n, 1e-10, dev.vp(out[:n]),
        dev.vp(out[n:2 * n]), dev.vp(out[2 * n:3 * n]), dev.vp(out[3 * n:4 * n]),
        dev.vp(out[4 * n:5 * n]), dev.vp(out[5 * n:6 * n]), dev.vp(out[6 * n:]),
        dev.vp(ints[4:6]), dev.vp(ints[0:1]), _st())
    _native.check(rc, "comparative")
    h = out.cpu().numpy()
    iv = ints.cpu().numpy()
    assert iv[0] == 0 and (iv[4], iv[5]) == (r, s)
    assert np.array_equal(h[:n], o_al) and np.array_equal(h[n:2 * n], o_be)
    rho, theta, p1, p2, d1, d2 = orc.comparative(o_al, o_be, r)
    assert np.array_equal(h[2 * n:3 * n], rho)
    assert np.max(np.abs(h[3 * n:4 * n] - theta)) <= 1e-15
    assert np.max(np.abs(h[4 * n:5 * n] - p1)) <= 1e-15
    assert abs(h[6 * n] - d1) <= 1e-14 and abs(h[6 * n + 1] - d2) <= 1e-14


@pytest.mark.parametrize("k,scale", [(60, 1e-8), (30, 3e-7), (64, 1e-10), (16, 0.0)])
def test_chol_inv_near_identity_path(k, scale):
    """Third CholeskyQR pass: Gram = I + E, |E| small -> expansion path; must
    equal the Cholesky inverse to fp64 roundoff."""
    kp = (k + 15) // 16 * 16
    rng = np.random.default_rng(k)
    x = rng.standard_normal((k, k))
    e = scale * (x + x.T)
    a = np.eye(k) + e
    G = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
    G[:k, :k] = torch.from_numpy(a)
    linv = torch.zeros(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
    rinv = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
    rd = torch.zeros(kp, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    _native.check(_native.lib().rgsv_chol_inv(dev.vp(G), k, kp, 0, dev.vp(linv), dev.vp(rinv),
                                              dev.vp(rd), dev.vp(status), _st()), "chol")
    li = linv[: kp * kp].view(kp, kp).cpu().numpy()
    ref = np.linalg.inv(np.linalg.cholesky(a))
    assert np.max(np.abs(li[:k, :k] - ref)) <= 1e-15
    assert np.array_equal(li[k:, k:], np.eye(kp - k)) and not np.any(li[:k, k:])
    assert np.max(np.abs(rd.cpu().numpy()[:k] - np.diag(np.linalg.cholesky(a)))) <= 1e-15
    assert np.array_equal(rinv.cpu().numpy(), li.T)


@pytest.mark.parametrize("rows,cols", [(60, 20), (20, 60), (128, 128), (300, 37)])
def test_core_svd_and_pseudoinverse_norm(rows, cols):
    """core.svd / core.pseudoinverse_norm (core.py:99-150) on the device
    Jacobi: reconstruction, orthonormal factors, LAPACK's singular values."""
    import paper_2404_09459_b200 as rg

    a = np.random.default_rng(rows * cols).standard_normal((rows, cols))
    f = rg.svd(a)
    r = min(rows, cols)
    assert f.u.shape == (rows, r) and f.s.shape == (r,) and f.v.shape == (cols, r)
    assert np.linalg.norm(f.u @ np.diag(f.s) @ f.v.T - a) <= 1e-12 * np.linalg.norm(a)
    assert np.linalg.norm(f.u.T @ f.u - np.eye(r)) <= 1e-12 * np.sqrt(r)
    assert np.linalg.norm(f.v.T @ f.v - np.eye(r)) <= 1e-12 * np.sqrt(r)
    s_ref = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(f.s - s_ref)) <= 1e-12 * s_ref[0]
    assert np.all(np.diff(f.s) <= 0)
    if rows >= cols:
        assert abs(rg.pseudoinverse_norm(a) - 1 / s_ref[-1]) <= 1e-10 / s_ref[-1]
    else:
        with pytest.raises(rg.RankDeficiencyError):
            rg.pseudoinverse_norm(a)
    b = a.copy()
    if rows >= cols:
        b[:, -1] = b[:, 0]
        with pytest.raises(rg.RankDeficiencyError):
            rg.pseudoinverse_norm(b)


@pytest.mark.parametrize("rows,kp", [(100000, 288), (5000, 208), (300, 144), (2000, 64),
                                     (20000, 192), (3001, 480)])
def test_gram_lower(rows, kp):
    """rgsv_gemm_gram_lower: the lower triangle of A^T A (the CholeskyQR
    Gram the blocked Cholesky reads) to fp64 accuracy; tiles strictly above
    the diagonal are skipped and left untouched."""
    rng = np.random.default_rng(rows + kp)
    a = rng.standard_normal((rows, kp))
    A = _dev(a)
    C = torch.full((kp, kp), 7.0, dtype=torch.float64, device="cuda")
    S = _scratch()
    _native.check(_native.lib().rgsv_gemm_gram_lower(dev.vp(A), A.stride(0), kp, rows, dev.vp(C),
                                                     kp, dev.vp(S), S.numel(), _st()), "gram")
    got = C.cpu().numpy()
    ref = a.T @ a
    low = np.tril_indices(kp)
    assert np.max(np.abs(got[low] - ref[low])) <= 1e-13 * np.abs(ref).max()
    up = got[np.triu_indices(kp, 1)]
    assert np.all((up == 7.0) | (np.abs(up - ref[np.triu_indices(kp, 1)]) <= 1e-9 * np.abs(ref).max()))
