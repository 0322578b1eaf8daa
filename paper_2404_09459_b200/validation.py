"""GmpPair rank validation on the device (reference engine.py:55-61).

The reference takes the singular values of vstack(G1, G2) with a dense
LAPACK SVD and keeps sigma_max and 1/sigma_min (engine.py:82-90). Here the
stacked pair is first reduced to its n x n triangular factor R -- the
singular values of [G1; G2] are those of R -- and R's singular values come
from the blocked one-sided Jacobi kernel:

* up to 1408 stacked rows: multi-CTA Householder QR (rgsv_dense_qr) straight
  from the two row sources (no stacked copy), rank-deficiency-safe;
* taller stacks with n <= 4096: shifted CholeskyQR3 and R = Q^T S (a
  CholeskyQR breakdown means cond > ~1e15, i.e. numerically rank deficient);
* n > 4096 (cfg4): DimensionError -- the check needs a 4096+ blocked
  Cholesky; build such pairs with check_rank=False.
"""

from __future__ import annotations

import torch

from . import device as _dev
from ._native import ST_JACOBI, check, lib
from .errors import ConvergenceError, DimensionError, RankDeficiencyError

MAX_CHECK_COLS = 4096


def _jacobi_values(a: torch.Tensor, rows: int, cols: int):
    sv = torch.zeros(min(rows, cols), dtype=torch.float64, device="cuda")
    ints = torch.zeros(4, dtype=torch.int32, device="cuda")
    ws_bytes = int(lib().rgsv_svd_values_workspace_bytes(rows, cols))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    rc = lib().rgsv_svd_values(_dev.vp(a), a.stride(0), rows, cols, _dev.vp(sv),
                               _dev.vp(ints[0:2]), _dev.vp(ints[2:3]), _dev.vp(ws), ws_bytes,
                               _dev.sp(torch.cuda.current_stream()))
    check(rc, "rgsv_svd_values")
    if int(ints[2].item()) & ST_JACOBI:
        raise ConvergenceError("Jacobi SVD did not converge")
    return sv.cpu().numpy()


def _f64(g: "_dev.DevMatrix") -> torch.Tensor:
    if not g.is_f32:
        return g.t
    t = torch.zeros((g.rows, g.cols + (g.cols & 1)), dtype=torch.float64, device="cuda")
    t[:, :g.cols].copy_(g.t)
    return t[:, :g.cols]


def can_check(g1: "_dev.DevMatrix", g2: "_dev.DevMatrix") -> bool:
    n = g1.cols
    return g1.rows + g2.rows <= 1408 or _dev.ceil16(n) <= MAX_CHECK_COLS


def stacked_r(g1: "_dev.DevMatrix", g2: "_dev.DevMatrix"):
    """The n x n triangular factor of [g1; g2] on the device, or None when
    CholeskyQR breaks down (numerically rank deficient stack)."""
    from .core import _gemm_at_b, _qr_in_place, dense_qr

    n = g1.cols
    rows = g1.rows + g2.rows
    a1, a2 = _f64(g1), _f64(g2)
    if rows <= 1408:
        _, r = dense_qr(a1, g1.rows, a2, g2.rows, n)
        return r
    if _dev.ceil16(n) > MAX_CHECK_COLS:
        raise DimensionError(f"the stacked-rank check supports n <= {MAX_CHECK_COLS} for "
                             f"{rows} stacked rows; build the pair with check_rank=False")
    kp = _dev.ceil16(n)
    y = torch.zeros((rows, kp), dtype=torch.float64, device="cuda")
    y[: g1.rows, :n].copy_(a1)
    y[g1.rows:, :n].copy_(a2)
    s0 = y.clone()
    try:
        _qr_in_place(y, rows, n, orig=s0)
    except RankDeficiencyError:
        return None
    return torch.triu(_gemm_at_b(y[:, :n], s0, n, n, rows))


def stacked_extreme_singular_values(g1: "_dev.DevMatrix", g2: "_dev.DevMatrix"):
    """(sigma_max, sigma_min) of vstack(g1, g2) (engine.py:55-57)."""
    n = g1.cols
    r = stacked_r(g1, g2)
    if r is None:
        return 1.0, 0.0
    # sigma_min <= min |R_jj| and sigma_max >= max |R_jj| for a triangular R:
    # a diagonal ratio at or below the threshold already proves the deficiency
    d = torch.diagonal(r[:n, :n]).abs()
    dmax, dmin = float(d.max()), float(d.min())
    if dmin <= 1e-12 * dmax:
        return dmax, dmin
    rr = torch.zeros((n, n + (n & 1)), dtype=torch.float64, device="cuda")
    rr[:, :n].copy_(r[:n, :n])
    s = _jacobi_values(rr, n, n)
    return float(s[0]), float(s[-1])
