"""Full GSVD factor recovery on the device (reference ``engine.py:278-362``).

``recover_gsvd`` rebuilds U (m x n), V (p x n) and R (n x n) with
G1 = U diag(alpha) R, G2 = V diag(beta) R from the compressed blocks
C1 = Q1ᵀG1, C2 = Q2ᵀG2 (or G1, G2 themselves for method="direct"):

* stacked QR  [C1; C2] = Q_S R̃           (shifted CholeskyQR3, Householder
                                            fallback; R̃ᵀ = Sᵀ Q_S by one GEMM)
* full SVD of the smaller L block        (rgsv_svd_vectors: one-sided Jacobi
                                            with accumulated rotations)
* U / V columns = Q_i · (singular vectors or L_j W)  (DMMA GEMMs)
* orthonormal completion of undetermined columns  (rgsv_orth_complete:
                                            columns of the complete Householder Q)
* R = Wᴴ R̃                               (DMMA GEMM)

All arithmetic runs in librgsv_b200.so; torch only allocates, slices and
flips buffers. Meaningful in the adaptive / direct regime, where
l1 + l2 >= n; the stacked width n is limited to 4096
(the blocked Cholesky; SVDs with vectors of 64+ vectors run on the blocked
multi-CTA Jacobi, completions beyond 1024 columns by projected CholeskyQR3).
"""

from __future__ import annotations

import dataclasses

import numpy as np
import torch

from . import device as _dev
from ._native import ST_CHOL, ST_JACOBI, check
from .errors import ConvergenceError, RecoveryError
from .rangefinder import _block_qr, _Ops, adaptive_device

F64 = torch.float64


def _buf(rows: int, cols: int) -> torch.Tensor:
    """Zeroed row-major device buffer with a 16-column-aligned pitch."""
    return torch.zeros((max(rows, 1), max(_dev.ceil16(cols), 16)), dtype=F64, device="cuda")


class _Dense:
    """Small dense helpers over the C-ABI (all operands row-major in HBM)."""

    def __init__(self):
        self.ops = _Ops()
        self.L = self.ops.L

    def st(self):
        return self.ops.st()

    def mm_bt(self, a, M: int, K: int, bt, N: int) -> torch.Tensor:
        """A (M x K) · Btᵀ with Bt (N x K)."""
        c = _buf(M, N)
        if M and N and K:
            self.ops.gx(_dev.vp(a), a.stride(0), _dev.vp(bt), bt.stride(0), _dev.vp(c),
                        c.stride(0), M, N, K)
        return c

    def at_b(self, a, K: int, M: int, b, N: int) -> torch.Tensor:
        """Aᵀ B with A (K x M), B (K x N)."""
        c = _buf(M, N)
        if M and N and K:
            self.ops.gtq(_dev.vp(a), a.stride(0), _dev.vp(b), b.stride(0), _dev.vp(c),
                         c.stride(0), M, N, K)
        return c

    def tr(self, a, rows: int, cols: int) -> torch.Tensor:
        """aᵀ (cols x rows)."""
        out = _buf(cols, rows)
        if rows and cols:
            check(self.L.rgsv_transpose(_dev.vp(out), out.stride(0), _dev.vp(a), a.stride(0),
                                        rows, cols, self.st()), "transpose")
        return out

    def complete(self, cols, dim: int, have: int, count: int) -> torch.Tensor:
        """`count` orthonormal columns orthogonal to cols[:, :have]
        (engine.py:278-291): np.eye(dim, count) when have == 0, else columns
        have..have+count of the complete Householder Q (one-CTA kernel, up to
        1024 columns each side), or beyond that a Gaussian block projected off
        cols twice and orthonormalized by shifted CholeskyQR3. Completion
        columns multiply classified-zero GSVs and are not determined by the
        data: any orthonormal completion is the reference's contract."""
        if have + count > dim:
            raise RecoveryError(f"cannot complete {have} columns with {count} more in "
                                f"dimension {dim}")
        out = _buf(dim, count)
        if count == 0:
            return out
        if have > 1024 or count > 1024:
            return self._complete_projected(cols, dim, have, count)
        a = _buf(dim, max(have, 1))
        if have:
            a[:dim, :have] = cols[:dim, :have]
        rd = torch.zeros(max(have, 1), dtype=F64, device="cuda")
        tau = torch.zeros(max(have, 1), dtype=F64, device="cuda")
        check(self.L.rgsv_orth_complete(_dev.vp(a), a.stride(0), dim, have, count, _dev.vp(out),
                                        out.stride(0), _dev.vp(rd), _dev.vp(tau), self.st()),
              "orth_complete")
        return out

    def _complete_projected(self, cols, dim: int, have: int, count: int) -> torch.Tensor:
        kp = _dev.ceil16(count)
        om = _dev.omega_device(dim, count, [0x5EED + have])[0]   # count x ldo (device)
        x = self.tr(om, count, dim)                              # dim x count
        x = x[:dim]
        for _ in range(2):                                       # x -= C (C^T x), twice
            t = self.at_b(cols, dim, have, x, count)             # have x count
            proj = self.mm_bt(cols, dim, have, self.tr(t, have, count), count)
            check(self.L.rgsv_axpy(_dev.vp(x), x.stride(0), _dev.vp(proj), proj.stride(0), dim,
                                   count, -1.0, self.st()), "axpy")
        y = torch.zeros((dim, kp), dtype=F64, device="cuda")
        y[:, :count] = x[:, :count]
        self.ops.status.zero_()
        q = self.ops.cholqr3(y, dim, count, kp)
        if int(self.ops.status.item()) & ST_CHOL:
            raise RecoveryError("orthonormal completion failed (CholeskyQR breakdown)")
        out = _buf(dim, count)
        out[:dim, :count] = q[:, :count]
        return out

    def scale_cols(self, a, rows: int, cols: int, d: torch.Tensor):
        if rows and cols:
            check(self.L.rgsv_scale_cols(_dev.vp(a), a.stride(0), rows, cols, _dev.vp(d),
                                         self.st()), "scale_cols")

    def svd_full(self, blk, rows: int, n: int):
        """np.linalg.svd(blk, full_matrices=True) restricted to what the
        recovery reads: (U[:, :min(rows, n)] (rows x min), Vh (n x n)),
        singular values descending; columns/rows for exactly-zero values are
        orthonormal completions."""
        status = torch.zeros(4, dtype=torch.int32, device="cuda")
        if rows <= n:  # vectors = the rows of blk
            nv, ln = rows, n
            v = _buf(nv, ln)
            v[:rows, :n] = blk[:rows, :n]
        else:  # vectors = the columns of blk
            nv, ln = n, rows
            v = self.tr(blk, rows, n)
        acc = _buf(nv, nv)
        jo = _buf(nv, nv)
        xn = _buf(nv, ln)
        sv = torch.zeros(nv, dtype=F64, device="cuda")
        if nv >= 64:  # blocked multi-CTA Jacobi with accumulated rotations
            nb = int(self.L.rgsv_svd_vectors_blocked_workspace_bytes(nv))
            ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
            check(self.L.rgsv_svd_vectors_blocked(
                _dev.vp(v), v.stride(0), nv, ln, _dev.vp(acc), acc.stride(0), _dev.vp(sv),
                _dev.vp(xn), xn.stride(0), _dev.vp(jo), jo.stride(0), 0, _dev.vp(status[1:2]),
                _dev.vp(status[0:1]), _dev.vp(ws), nb, self.st()), "svd_vectors_blocked")
        else:
            check(self.L.rgsv_svd_vectors(_dev.vp(v), v.stride(0), nv, ln, _dev.vp(acc),
                                          acc.stride(0), _dev.vp(sv), _dev.vp(xn), xn.stride(0),
                                          _dev.vp(jo), jo.stride(0), 0, _dev.vp(status[1:2]),
                                          _dev.vp(status[0:1]), self.st()), "svd_vectors")
        code, nzero = (int(x) for x in status[:2].cpu().tolist())
        if code & ST_JACOBI:
            raise ConvergenceError("Jacobi SVD of an L block did not converge")
        self.last_sv = sv  # descending singular values (core.svd reads them)
        if rows <= n:
            u = self.tr(jo, nv, nv)                      # U = Jᵀ (rows x rows)
            vh = _buf(n, n)
            have = rows - nzero
            vh[:have, :n] = xn[:have, :n]
            if have < n:                                 # complete the row space
                xt = self.tr(xn, have, n) if have else _buf(n, 1)
                comp = self.complete(xt, n, have, n - have)
                vh[have:n, :n] = self.tr(comp, n, n - have)[: n - have, :n]
            return u, vh
        u = self.tr(xn, n, rows)                         # U = Xᵀ (rows x n)
        if nzero:
            have = n - nzero
            comp = self.complete(u, rows, have, nzero)
            u[:rows, have:n] = comp[:rows, :nzero]
        return u, jo                                     # Vh = J (n x n)


def _flip_rows(t: torch.Tensor, rows: int, cols: int) -> torch.Tensor:
    out = _buf(rows, cols)
    out[:rows, :cols] = torch.flip(t[:rows, :cols], dims=(0,))
    return out


def _flip_cols(t: torch.Tensor, rows: int, cols: int) -> torch.Tensor:
    out = _buf(rows, cols)
    out[:rows, :cols] = torch.flip(t[:rows, :cols], dims=(1,))
    return out


def recover(pair, opts, direct: bool):
    """engine.py:294-362 on the device; returns (u, v, r_factor, spectrum)."""
    from .engine import GsvSpectrum, _spectrum_checked

    m, p, n = pair.m, pair.p, pair.n
    if m < n or p < n:
        raise RecoveryError(f"full recovery needs m >= n and p >= n, got ({m}, {p}, {n})")
    if direct:
        c1, c2 = pair.g1.t, pair.g2.t
        l1, l2 = m, p
        q1 = q2 = None
    else:
        cfg = opts.extraction
        q1, c1, _ = adaptive_device(pair.g1, cfg)
        q2, c2, _ = adaptive_device(pair.g2, dataclasses.replace(cfg, seed=cfg.seed + 1))
        l1, l2 = c1.shape[0], c2.shape[0]
    l = l1 + l2
    if min(l, n) != n:                                   # engine.py:309-313
        raise RecoveryError("compressed pair has fewer than n independent columns; "
                            "tighten the extraction tolerance")
    if n > 4096:
        raise RecoveryError(f"device recovery supports n <= 4096, got n={n}")
    spec: GsvSpectrum = _spectrum_checked(c1, l1, c2, l2, n, opts.classify_tol)
    alphas, betas, r, s = spec.alphas, spec.betas, spec.r, spec.s
    tol = opts.classify_tol
    D = _Dense()
    kpn = _dev.ceil16(n)
    # stacked QR with its R factor (engine.py:257)
    S = torch.zeros((l, kpn), dtype=F64, device="cuda")
    if l1:
        S[:l1, :n] = c1[:l1, :n]
    if l2:
        S[l1:, :n] = c2[:l2, :n]
    qs, _ = _block_qr(D.ops, S, l, n, kpn, 0.0)
    rt_t = D.at_b(S, l, n, qs, n)                        # R̃ᵀ = Sᵀ Q_S
    rt_t[:n, :n] = torch.tril(rt_t[:n, :n])
    l1b = qs[:l1] if l1 else None
    l2b = qs[l1:] if l2 else None

    if l1 <= l2:                                         # engine.py:321-338
        u1, w1h = D.svd_full(l1b, l1, n)
        ncols = min(l1, n)
        u_main = u1 if q1 is None else D.mm_bt(q1, m, l1, D.tr(u1, l1, ncols), ncols)
        u = _buf(m, n)
        u[:m, :ncols] = u_main[:m, :ncols]
        if n > ncols:
            u[:m, ncols:n] = D.complete(u_main, m, ncols, n - ncols)[:m, : n - ncols]
        t_t = D.mm_bt(w1h, n, n, l2b, l2)                # (L2 W1)ᵀ
        v_raw = D.tr(t_t, n, l2) if q2 is None else D.mm_bt(q2, p, l2, t_t, n)
        if np.any(betas[r:] < tol):
            raise RecoveryError("interior GSV below classify_tol; recovery ill conditioned")
        v = _buf(p, n)
        v[:p, r:n] = v_raw[:p, r:n]
        dv = torch.from_numpy(np.ascontiguousarray(betas[r:])).to("cuda")
        D.scale_cols(v[:, r:], p, n - r, dv)
        if r:
            vr = _buf(p, n - r)
            vr[:p, : n - r] = v[:p, r:n]
            v[:p, :r] = D.complete(vr, p, n - r, r)[:p, :r]
        rf = D.mm_bt(w1h, n, n, rt_t, n)                 # W1ᴴ R̃
    else:                                                # engine.py:339-360
        u2, w2h = D.svd_full(l2b, l2, n)
        nvals = min(l2, n)
        w2 = _flip_rows(w2h, n, n)
        v_block = _flip_cols(u2, l2, nvals)
        v_main = v_block if q2 is None else D.mm_bt(q2, p, l2, D.tr(v_block, l2, nvals), nvals)
        v = _buf(p, n)
        v[:p, n - nvals:n] = v_main[:p, :nvals]
        if n > nvals:
            v[:p, : n - nvals] = D.complete(v_main, p, nvals, n - nvals)[:p, : n - nvals]
        t_t = D.mm_bt(w2, n, n, l1b, l1)                 # (L1 W2ᴴᵀ)ᵀ
        u_raw = D.tr(t_t, n, l1) if q1 is None else D.mm_bt(q1, m, l1, t_t, n)
        nz = r + s
        if np.any(alphas[:nz] < tol):
            raise RecoveryError("interior GSV below classify_tol; recovery ill conditioned")
        u = _buf(m, n)
        u[:m, :nz] = u_raw[:m, :nz]
        da = torch.from_numpy(np.ascontiguousarray(alphas[:nz])).to("cuda")
        D.scale_cols(u, m, nz, da)
        if n > nz:
            u[:m, nz:n] = D.complete(u, m, nz, n - nz)[:m, : n - nz]
        rf = D.mm_bt(w2, n, n, rt_t, n)                  # w2 R̃
    return (u[:m, :n].cpu().numpy(), v[:p, :n].cpu().numpy(), rf[:n, :n].cpu().numpy(), spec)


__all__ = ["recover"]
