"""Matrix primitives of the drop-in API (reference ``rgsv/core.py``).

``gaussian_matrix`` keeps the reference's seeded host generator (PCG64 via
``numpy.random.default_rng``, core.py:60-76) because the sketches must use
the reference's own Ω; everything that touches the matrices themselves
runs on the B200 (``frobenius_norm``/``sum_sq`` through the device
sum-of-squares kernel, ``reduced_qr`` through shifted CholeskyQR3).
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


def reduced_qr(m) -> QrFactors:
    """Reduced QR of a tall full-column-rank matrix (cols <= 1024) by shifted
    CholeskyQR3 on the B200; R has a positive diagonal, which is the
    reference's phase convention (core.py:79-96)."""
    g = as_matrix(m)
    rows, cols = g.rows, g.cols
    if rows < cols:
        raise DimensionError("B200 reduced_qr supports tall matrices (rows >= cols)")
    kp = _dev.ceil16(cols)
    if kp > 1024:
        raise DimensionError("B200 reduced_qr supports at most 1024 columns")
    y = torch.zeros((rows, kp), dtype=torch.float64, device="cuda")
    y[:, :cols].copy_(g.t[:, :cols])
    r = _qr_in_place(y, rows, cols)
    return QrFactors(y[:, :cols].cpu().numpy(), r[:cols, :cols].cpu().numpy())


def _qr_in_place(y: torch.Tensor, rows: int, k: int) -> torch.Tensor:
    """CholQR3 on the device through the C-ABI building blocks; y (rows x kp)
    is replaced by Q, returns R (kp x kp) = R3 R2 R1."""
    L = lib()
    kp = y.shape[1]
    st = _dev.sp(torch.cuda.current_stream())
    gram = torch.empty((kp, kp), dtype=torch.float64, device="cuda")
    linv = torch.empty(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
    rinv = torch.empty((kp, kp), dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    scratch = torch.empty(148 * kp * max(kp, 128) + 4096, dtype=torch.float64, device="cuda")
    tmp = torch.empty_like(y)
    r_acc = torch.eye(kp, dtype=torch.float64, device="cuda")
    src, dst = y, tmp
    for step in range(3):
        check(L.rgsv_gemm_gtq(_dev.vp(src), kp, _dev.vp(src), kp, _dev.vp(gram), kp, kp, kp, rows,
                              _dev.vp(scratch), scratch.numel() * 8, st), "gram")
        check(L.rgsv_chol_inv(_dev.vp(gram), k, kp, rows if step == 0 else 0, _dev.vp(linv),
                              _dev.vp(rinv), None, _dev.vp(status), st), "chol")
        check(L.rgsv_gemm_gx(_dev.vp(src), kp, _dev.vp(linv), kp, _dev.vp(dst), kp, rows, kp, kp,
                             _dev.vp(scratch), scratch.numel() * 8, st), "trsm")
        # R_step = (Rinv)^-1 accumulated on the device: R_acc <- R_step R_acc
        rstep = torch.linalg.solve_triangular(rinv, torch.eye(kp, dtype=torch.float64,
                                                              device="cuda"), upper=True)
        r_acc = rstep @ r_acc
        src, dst = dst, src
    if int(status.item()) != 0:
        from .errors import RankDeficiencyError

        raise RankDeficiencyError("CholeskyQR breakdown: matrix is numerically rank deficient")
    if src is not y:
        y.copy_(src)
    return r_acc


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
    if min(rows, cols) > 2048:
        raise DimensionError("B200 svd supports min(rows, cols) <= 2048 (one-sided Jacobi)")
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
        if _dev.ceil16(cols) > 1024:
            raise
        y = torch.zeros((rows, _dev.ceil16(cols)), dtype=torch.float64, device="cuda")
        y[:, :cols] = g.t
        r = _qr_in_place(y, rows, cols)[:cols, :cols].contiguous()  # raises RankDeficiencyError
        sv = _jacobi_values(r, cols, cols)
    smax, smin = float(sv[0]), float(sv[-1])
    if smin <= 1e-13 * smax:
        raise RankDeficiencyError(f"smallest singular value {smin:.3e} below rank threshold "
                                  f"{1e-13 * smax:.3e}")
    return 1.0 / smin
