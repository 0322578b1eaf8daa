"""Matrix primitives of the drop-in API (reference ``rgsv/core.py``).

``gaussian_matrix`` keeps the reference's seeded host generator (PCG64 via
``numpy.random.default_rng``, core.py:60-76) because the sketches must use
the reference's own Ω; everything that touches the matrices themselves
runs on the B200 (``frobenius_norm``/``sum_sq`` through the device
sum-of-squares kernel, ``reduced_qr`` through the multi-CTA Householder
kernel or shifted CholeskyQR3). No cuBLAS/cuSOLVER call is made.
"""

from __future__ import annotations

import math
from typing import NamedTuple

import numpy as np
import torch

from . import device as _dev
from ._native import check, lib
from .errors import ConvergenceError, DimensionError, RankDeficiencyError, ValidationError

REAL = "real"
COMPLEX = "complex"
_SEED_MASK = (1 << 64) - 1


class QrFactors(NamedTuple):
    """Reduced QR factors (core.py:25-31): q orthonormal columns, r upper
    triangular with nonnegative diagonal."""

    q: np.ndarray
    r: np.ndarray


class SvdFactors(NamedTuple):
    """Reduced SVD factors (core.py:34-40)."""

    u: np.ndarray
    s: np.ndarray
    v: np.ndarray


def as_matrix(a, name: str = "matrix"):
    """Validate a 2-D nonempty real matrix and place it in HBM (core.py:43-57).
    Returns a ``DevMatrix``; non-finite entries are rejected on the device."""
    g = _dev.to_device(a, name)
    ss = _dev.device_sumsq(g)
    if not math.isfinite(ss):
        raise ValidationError(f"{name} contains non-finite entries")
    return g


def gaussian_matrix(rows: int, cols: int, seed: int, field: str = REAL) -> np.ndarray:
    """Bitwise-reproducible Gaussian matrix, reference convention
    (core.py:60-76)."""
    if rows < 1 or cols < 1:
        raise DimensionError(f"matrix dimensions must be positive, got ({rows}, {cols})")
    rng = np.random.default_rng(int(seed) & _SEED_MASK)
    if field == REAL:
        return rng.standard_normal((rows, cols))
    if field == COMPLEX:
        re = rng.standard_normal((rows, cols))
        im = rng.standard_normal((rows, cols))
        return math.sqrt(0.5) * (re + 1j * im)
    raise ValidationError(f"field must be 'real' or 'complex', got {field!r}")


def sum_sq(a) -> float:
    """Sum of squared entries, computed on the device (core.py:115-125)."""
    return _dev.device_sumsq(_dev.to_device(a))


def frobenius_norm(m) -> float:
    """Frobenius norm on the device (core.py:128-130)."""
    return math.sqrt(sum_sq(as_matrix(m)))


HH_MAX_ROWS = 1408  # rgsv_dense_qr (multi-CTA Householder) row limit
CHOL_MAX_COLS = 4096  # blocked-Cholesky limit of the CholeskyQR3 route


def reduced_qr(m) -> QrFactors:
    """Reduced QR with the reference's phase convention diag(R) >= 0
    (core.py:79-96), tall or wide, on the B200:

    * rows <= 1408: blocked Householder over many CTAs (rgsv_dense_qr), the
      LAPACK dgeqrf/dorgqr algorithm numpy.linalg.qr runs; rank deficiency
      is permitted exactly as in the reference (R_jj ~ 0);
    * taller matrices (cols <= 4096): shifted CholeskyQR3, R = Q^T A; a
      CholeskyQR breakdown (numerical rank deficiency) falls back to the
      one-CTA Householder kernel (cols <= 1024);
    * wide matrices with more than 1408 rows: CholeskyQR3 of the leading
      rows x rows block (rows <= 4096), R = Q^T A.
    """
    g = as_matrix(m)
    rows, cols = g.rows, g.cols
    if rows <= HH_MAX_ROWS:
        q, r = dense_qr(g.t, rows, None, 0, cols)
        return QrFactors(q.cpu().numpy(), r.cpu().numpy())
    if rows >= cols:
        if _dev.ceil16(cols) > CHOL_MAX_COLS:
            raise DimensionError(f"B200 reduced_qr supports at most {CHOL_MAX_COLS} columns")
        q, r = tall_qr(g.t, rows, cols)
        return QrFactors(q.cpu().numpy(), r.cpu().numpy())
    if _dev.ceil16(rows) > CHOL_MAX_COLS:
        raise DimensionError(f"B200 reduced_qr of a wide matrix supports at most "
                             f"{CHOL_MAX_COLS} rows")
    q, _ = tall_qr(g.t[:, :rows], rows, rows)
    r = _gemm_at_b(q, g.t, rows, cols, rows)
    return QrFactors(q.cpu().numpy(), torch.triu(r).cpu().numpy())


def dense_qr(a1: torch.Tensor, m1: int, a2, m2: int, n: int, want_r: bool = True,
             phase_fix: bool = True):
    """Householder QR of the row stack [a1 (m1 rows); a2 (m2 rows)] (device
    tensors, fp64, m1 + m2 <= 1408): Q (M x K) and R (K x n) tensors,
    K = min(M, n) -- rgsv_dense_qr, one cooperative launch."""
    L = lib()
    M = m1 + m2
    K = min(M, n)
    q = torch.empty((M, K), dtype=torch.float64, device="cuda")
    r = torch.empty((K, n), dtype=torch.float64, device="cuda") if want_r else None
    nb = int(L.rgsv_dense_qr_workspace_bytes(M, n))
    if nb == 0:
        raise DimensionError(f"Householder QR supports at most {HH_MAX_ROWS} rows, got {M}")
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    st = _dev.sp(torch.cuda.current_stream())
    check(L.rgsv_dense_qr(_dev.vp(a1), a1.stride(0), m1, _dev.vp(a2) if a2 is not None else None,
                          a2.stride(0) if a2 is not None else 0, m2, n, _dev.vp(q), K,
                          _dev.vp(r) if r is not None else None, n if r is not None else 0,
                          1 if phase_fix else 0, _dev.vp(ws), nb, st), "rgsv_dense_qr")
    return q, r


def _scratch_for(kp: int) -> torch.Tensor:
    """Split-K partial storage for the GEMMs of a kp-wide CholeskyQR: tail
    tiles of the G X passes (<= 148 x 128 rows) or a few kp x kp Gram
    partials, whichever is larger."""
    return torch.empty(max(148 * 128 * max(kp, 128), 4 * kp * kp) + 4096, dtype=torch.float64,
                       device="cuda")


def _gemm_at_b(a: torch.Tensor, b: torch.Tensor, m_out: int, n_out: int, rows: int):
    """C (m_out x n_out) = A^T B over `rows` rows (rgsv_gemm_gtq, DMMA)."""
    L = lib()
    c = torch.empty((m_out, n_out + (n_out & 1)), dtype=torch.float64, device="cuda")
    scratch = _scratch_for(_dev.ceil16(max(m_out, 16)))
    check(L.rgsv_gemm_gtq(_dev.vp(a), a.stride(0), _dev.vp(b), b.stride(0), _dev.vp(c),
                          c.stride(0), m_out, n_out, rows, _dev.vp(scratch),
                          scratch.numel() * 8, _dev.sp(torch.cuda.current_stream())), "gtq")
    return c[:, :n_out]


def tall_qr(a: torch.Tensor, rows: int, cols: int):
    """Reduced QR of a tall device matrix (rows x cols view, fp64): shifted
    CholeskyQR3 (R = Q^T A, diag > 0), or -- when CholeskyQR breaks down on
    a numerically rank-deficient matrix -- the one-CTA Householder kernel
    with the reference's phase fix. Returns (Q rows x cols, R cols x cols)."""
    kp = _dev.ceil16(cols)
    y = torch.zeros((rows, kp), dtype=torch.float64, device="cuda")
    y[:, :cols].copy_(a[:, :cols])
    try:
        _qr_in_place(y, rows, cols, orig=a)
        q = y[:, :cols]
        r = torch.triu(_gemm_at_b(q, a, cols, cols, rows))
        d = torch.diagonal(r).abs()
        # shifted CholeskyQR3 is accurate up to cond ~ 1/u; a (near) rank
        # deficient matrix (the shift keeps the Cholesky alive) goes to the
        # Householder kernel, which reproduces LAPACK's R_jj ~ 0
        if kp > 1024 or float(d.min()) > 1e-10 * float(d.max()):
            return q, r
        raise RankDeficiencyError("near rank deficient")
    except RankDeficiencyError:
        if kp > 1024:
            raise
        L = lib()
        w = y.clone()
        w[:, :cols].copy_(a[:, :cols])
        w[:, cols:] = 0.0
        qq = torch.zeros((rows, kp), dtype=torch.float64, device="cuda")
        rd = torch.zeros(kp, dtype=torch.float64, device="cuda")
        tau = torch.zeros(kp, dtype=torch.float64, device="cuda")
        check(L.rgsv_householder_qr(_dev.vp(w), kp, rows, cols, _dev.vp(qq), kp, _dev.vp(rd),
                                    _dev.vp(tau), _dev.sp(torch.cuda.current_stream())),
              "householder_qr")
        q = qq[:, :cols]
    r = _gemm_at_b(q, a, cols, cols, rows)
    return q, torch.triu(r)


def _qr_in_place(y: torch.Tensor, rows: int, k: int, orig: torch.Tensor | None = None) -> None:
    """Shifted CholeskyQR3 on the device through the C-ABI building blocks;
    y (rows x kp) is replaced by Q. RankDeficiencyError on breakdown.

    Shifted CholeskyQR3 needs cond(Q1)^2 * n * u < 1 for its unshifted second
    pass, which fails from cond(Y) ~ 1e10 at n ~ 1000 although Y has full
    numerical rank (the reference accepts stacks up to 1e12, engine.py:57).
    With ``orig`` (the untouched input) a breakdown is retried with a second
    shifted pass, shift / shift / plain / plain: each shifted pass takes the
    condition number down by ~sqrt(shift), so the plain passes see
    cond <~ 1e5 for any input up to ~1/u. A genuinely rank-deficient matrix
    still breaks down in the plain passes and raises."""
    L = lib()
    kp = y.shape[1]
    st = _dev.sp(torch.cuda.current_stream())
    gram = torch.empty((kp, kp), dtype=torch.float64, device="cuda")
    linv = torch.empty(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    scratch = _scratch_for(kp)
    tmp = torch.empty_like(y)

    def passes(shifts) -> bool:
        src, dst = y, tmp
        for shift_rows in shifts:
            check(L.rgsv_gemm_gtq(_dev.vp(src), kp, _dev.vp(src), kp, _dev.vp(gram), kp, kp, kp,
                                  rows, _dev.vp(scratch), scratch.numel() * 8, st), "gram")
            check(L.rgsv_chol_inv(_dev.vp(gram), k, kp, shift_rows, _dev.vp(linv), None, None,
                                  _dev.vp(status), st), "chol")
            check(L.rgsv_gemm_gx(_dev.vp(src), kp, _dev.vp(linv), kp, _dev.vp(dst), kp, rows, kp,
                                 kp, _dev.vp(scratch), scratch.numel() * 8, st), "trsm")
            src, dst = dst, src
        if int(status.item()) != 0:
            return False
        if src is not y:
            y.copy_(src)
        return True

    if passes((rows, 0, 0)):
        return
    if orig is not None:
        y.zero_()
        y[:, :k].copy_(orig[:, :k])
        status.zero_()
        if passes((rows, rows, 0, 0)):
            return
    raise RankDeficiencyError("CholeskyQR breakdown: matrix is numerically rank deficient")


__all__ = ["REAL", "COMPLEX", "QrFactors", "SvdFactors", "as_matrix", "gaussian_matrix",
           "sum_sq", "frobenius_norm", "reduced_qr"]


def svd(m) -> SvdFactors:
    """Reduced SVD (core.py:99-106) on the device: one-sided Jacobi with
    accumulated rotations (rgsv_svd_vectors), orthonormal completion for
    exactly-zero singular values; ``u @ diag(s) @ v.T`` reconstructs the
    input, ``s`` nonincreasing. Non-convergence raises ConvergenceError
    (the reference's LinAlgError mapping)."""
    from .recovery import _buf, _Dense

    g = as_matrix(m)
    rows, cols = g.rows, g.cols
    if min(rows, cols) > 8192:
        raise DimensionError("B200 svd supports min(rows, cols) <= 8192 (blocked Jacobi)")
    blk = _buf(rows, cols)
    blk[:rows, :cols] = g.t
    dense = _Dense()
    u, vh = dense.svd_full(blk, rows, cols)
    r = min(rows, cols)
    s = dense.last_sv[:r]
    if rows <= cols:
        u_red, v_red = u[:rows, :r], vh[:r, :cols].T
    else:
        u_red, v_red = u[:rows, :r], vh[:cols, :cols].T
    return SvdFactors(u_red.cpu().numpy(), s.cpu().numpy(), v_red.cpu().numpy())


def pseudoinverse_norm(m) -> float:
    """1 / sigma_min for a matrix of full column rank (core.py:133-150);
    singular values from the device Jacobi. RankDeficiencyError otherwise."""
    from .validation import _jacobi_values

    g = as_matrix(m)
    rows, cols = g.rows, g.cols
    if rows < cols:
        raise RankDeficiencyError(f"matrix of shape {(rows, cols)} cannot have full column rank")
    a = torch.zeros((rows, cols + (cols & 1)), dtype=torch.float64, device="cuda")
    a[:, :cols] = g.t
    try:
        sv = _jacobi_values(a, rows, cols)
    except ConvergenceError:
        # exactly dependent columns can stall the values-only Jacobi; the
        # CholeskyQR route then reports the rank deficiency like the reference
        if _dev.ceil16(cols) > CHOL_MAX_COLS:
            raise
        y = torch.zeros((rows, _dev.ceil16(cols)), dtype=torch.float64, device="cuda")
        y[:, :cols] = g.t
        _qr_in_place(y, rows, cols, orig=g.t)  # raises RankDeficiencyError
        r = _gemm_at_b(y[:, :cols], g.t, cols, cols, rows)
        sv = _jacobi_values(torch.triu(r).contiguous(), cols, cols)
    smax, smin = float(sv[0]), float(sv[-1])
    if smin <= 1e-13 * smax:
        raise RankDeficiencyError(f"smallest singular value {smin:.3e} below rank threshold "
                                  f"{1e-13 * smax:.3e}")
    return 1.0 / smin
