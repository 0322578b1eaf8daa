"""GmpPair rank validation on the device (reference engine.py:55-61).

The reference takes the singular values of vstack(G1, G2) with a dense
LAPACK SVD. Here the singular values come from one-sided Jacobi on the
device: directly on the stacked matrix when it is small, otherwise on the
R factor of a shifted CholeskyQR3 of the stacked pair (same singular
values; n <= 1024, the blocked Cholesky limit).
"""

from __future__ import annotations

import torch

from . import device as _dev
from ._native import ST_JACOBI, check, lib
from .errors import ConvergenceError, DimensionError, RankDeficiencyError

_DIRECT_LIMIT = 1 << 22  # entries of the stacked matrix handled by direct Jacobi


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


def stacked_extreme_singular_values(g1: "_dev.DevMatrix", g2: "_dev.DevMatrix"):
    n = g1.cols
    rows = g1.rows + g2.rows
    if rows * n <= _DIRECT_LIMIT:
        stacked = torch.empty((rows, n + (n & 1)), dtype=torch.float64, device="cuda")
        stacked[: g1.rows, :n].copy_(g1.t)
        stacked[g1.rows:, :n].copy_(g2.t)
        s = _jacobi_values(stacked, rows, n)
        return float(s[0]), float(s[-1])
    from .core import _qr_in_place

    kp = _dev.ceil16(n)
    if kp > 1024:
        raise DimensionError("check_rank supports n <= 1024 for large stacked pairs")
    y = torch.zeros((rows, kp), dtype=torch.float64, device="cuda")
    y[: g1.rows, :n].copy_(g1.t)
    y[g1.rows:, :n].copy_(g2.t)
    try:
        r = _qr_in_place(y, rows, n)
    except RankDeficiencyError:
        return 1.0, 0.0
    r = r[:n, :n].contiguous()
    s = _jacobi_values(r, n, n)
    return float(s[0]), float(s[-1])
