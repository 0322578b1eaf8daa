"""fp32-resident pairs on the 5th-gen tensor cores (the cfg4 family).

The G passes of the fixed-rank chain -- sketch Y = G Omega
(rangefinder.py:115), the q power steps Z = G^T Q / Y = G Qhat, and the
projection B = Q^T G (engine.py:255-256) -- run as tcgen05 kind::tf32 GEMMs
with a 3xTF32 hi/lo operand split (csrc/tf32x3.cu): fp32-level products at
three TF32 MMAs each, fp32 accumulation in TMEM, fp64 outputs. The small
factorizations (shifted CholeskyQR3 of Y and Z, the stacked QR, Jacobi and
the comparative kernel) stay fp64 on the DMMA path.

The reference promotes fp32 input to fp64 up front (core.py:51-54); the
promoted chain (rangefinder.chunked_chain) reproduces that exactly and stays
available as GsvOptions(f32_mode="promote"). This module is the fp32
compute path BASELINE.json's cfg4 asks for (tolerance 1e-4 on the GSVs and
theta); tests/test_gpu_tf32.py pins it against the fp64 oracle.
"""

from __future__ import annotations

import math

import torch

from . import device as _dev
from ._native import check, lib
from .errors import RankDeficiencyError, ValidationError

F32, F64 = torch.float32, torch.float64
ST_CHOL = 0x1

# How the tensor core reads the low 13 mantissa bits of a raw fp32 operand
# (0: dropped, 1: rounded to nearest); lo = tf32(g - hi(g)) must use the same
# hi. Measured on B200 by tests/test_gpu_tf32.py::test_tc_reads_fp32_as.
HI_MODE = 0


def _ceil(x: int, m: int) -> int:
    return (x + m - 1) // m * m


class TF32Ops:
    """Launch helpers on the current stream (scratch owned here)."""

    def __init__(self):
        self.L = lib()
        self.scratch = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
        self.ws = torch.empty(4096, dtype=F64, device="cuda")

    @staticmethod
    def st():
        return _dev.sp(torch.cuda.current_stream())

    def split_big(self, g: "_dev.DevMatrix", lo: torch.Tensor | None = None):
        """(lo, ||G||_F^2 as a device scalar) for an fp32 DevMatrix."""
        if lo is None:
            lo = torch.empty((g.rows, g.ld), dtype=F32, device="cuda")
        ss = torch.zeros(1, dtype=F64, device="cuda")
        check(self.L.rgsv_f32_split(_dev.vp(g.t), g.ld, g.rows, g.cols, _dev.vp(lo), lo.stride(0),
                                    HI_MODE, _dev.vp(ss), _dev.vp(self.ws), self.ws.numel() * 8,
                                    self.st()), "f32_split")
        return lo, ss

    def split_small(self, x: torch.Tensor, rows: int, cols: int, cols_out: int,
                    rows_out: int | None = None):
        """hi/lo fp32 (rows_out x cols_out, zero padded) of an fp64 matrix x
        (rows x cols)."""
        ro = rows_out or rows
        alloc = torch.zeros if ro > rows else torch.empty
        hi = alloc((ro, cols_out), dtype=F32, device="cuda")
        lo = alloc((ro, cols_out), dtype=F32, device="cuda")
        check(self.L.rgsv_f64_split_tf32(_dev.vp(x), x.stride(0), rows, cols, _dev.vp(hi),
                                         _dev.vp(lo), cols_out, cols_out, self.st()),
              "f64_split_tf32")
        return hi, lo

    def gx(self, g, glo, xhi, xlo, y, M: int, N: int, K: int):
        """y (M x N fp64) = G (M x K) X^T."""
        check(self.L.rgsv_tf32x3_gx(_dev.vp(g.t), _dev.vp(glo), g.ld, _dev.vp(xhi), _dev.vp(xlo),
                                    xhi.stride(0), _dev.vp(y), y.stride(0), M, N, K, self.st()),
              "tf32x3_gx")

    def gtq(self, qhi, qlo, g, glo, out, N: int, M: int, K: int):
        """out (N x M fp64) = Q^T G (split-K partials in scratch, grown on demand)."""
        while True:
            rc = self.L.rgsv_tf32x3_gtq(_dev.vp(qhi), _dev.vp(qlo), qhi.stride(0), _dev.vp(g.t),
                                        _dev.vp(glo), g.ld, _dev.vp(out), out.stride(0), N, M, K,
                                        _dev.vp(self.scratch), self.scratch.numel(), self.st())
            if rc != 6:  # RGSV_ERR_WORKSPACE
                return check(rc, "tf32x3_gtq")
            self.scratch = torch.empty(self.scratch.numel() * 4, dtype=torch.uint8, device="cuda")


def supported(g: "_dev.DevMatrix", k: int) -> bool:
    """Shapes served by the tf32x3 kernels (else the promoted fp64 chain)."""
    kq = _ceil(_dev.ceil16(k), 32)
    return g.is_f32 and g.ld % 4 == 0 and g.t.data_ptr() % 16 == 0 and kq <= 320 and \
        g.cols >= 1 and g.rows >= 1


def _noreduce(x):
    return x


def cholqr_mixed(ops, t: TF32Ops, y: torch.Tensor, m: int, k: int, kp: int, final: bool,
                 reduce=_noreduce, rows_total: int | None = None):
    """Shifted CholeskyQR for the fp32 chain (m x kp fp64 Y -> Q, zero padded).

    Pass 1: fp64 Gram (shifted) and Cholesky -- the Gram's condition is
    cond(Y)^2, beyond fp32 -- with the TRSM Y L^-T on the tensor cores
    (3xTF32). Pass 2: 3xTF32 Gram and TRSM of the now well-conditioned Q1.
    Pass 3 (final basis only): fp64 Gram, Cholesky and TRSM, so the returned
    Q is orthonormal to fp64 precision. Every factor is triangular, so the
    nested leading spans are those of Y (the intermediate basis of a power
    step only needs its span: two passes). For a row-sharded Y (dist.py)
    `reduce` all-reduces each k x k Gram and `rows_total` sets the shift."""
    kq = _ceil(kp, 32)
    f64 = torch.float64

    def trsm_tc(src_hi, src_lo, linv):
        xh, xl = t.split_small(linv, kp, kp, kp, rows_out=kq)
        out = torch.empty((m, kq), dtype=f64, device="cuda")
        t.gx(_dev.DevMatrix(src_hi[:, :kp], m, kp), src_lo, xh, xl, out, m, kq, kp)
        return out

    # pass 1
    gram = torch.zeros((kp, kp), dtype=f64, device="cuda")
    ops.gram(_dev.vp(y), kp, kp, m, _dev.vp(gram))
    linv, _ = ops.chol(reduce(gram), k, kp, rows_total or m)
    yh, yl = t.split_small(y, m, kp, kp)
    q1 = trsm_tc(yh, yl, linv)
    del yh, yl
    # pass 2
    qh, ql = t.split_small(q1, m, kp, kq)
    g2 = torch.zeros((kq, kq), dtype=f64, device="cuda")
    t.gtq(qh, ql, _dev.DevMatrix(qh[:, :kp], m, kp), ql, g2, kq, kp, m)
    linv2, _ = ops.chol(reduce(g2[:kp, :kp].contiguous()), k, kp, 0)
    q2 = trsm_tc(qh, ql, linv2)
    del qh, ql, q1
    q2 = q2 if kq == kp else q2[:, :kp].contiguous()
    if not final:
        return q2
    # pass 3: fp64 Gram and Cholesky. Q2 is orthonormal to ~1e-6, so
    # L3^-1 = I + D with |D| ~ 1e-6, and the TRSM Q = Q2 L3^-T is computed as
    # Q2 + Q2 D^T: the small correction on the tensor cores (3xTF32: ~1e-13
    # absolute error), the identity part exact in fp64 -- the fp64 DMMA TRSM
    # took 6.9 ms on cfg4's 1e6 x 288 Y.
    gram3 = torch.zeros((kp, kp), dtype=f64, device="cuda")
    ops.gram(_dev.vp(q2), kp, kp, m, _dev.vp(gram3))
    linv3, _ = ops.chol(reduce(gram3), k, kp, 0)
    eye = torch.eye(kp, dtype=f64, device="cuda")
    check(ops.L.rgsv_axpy(_dev.vp(linv3), kp, _dev.vp(eye), kp, kp, kp, -1.0, ops.st()),
          "axpy")  # D = L3^-1 - I
    q2h, q2l = t.split_small(q2, m, kp, kp)
    corr = trsm_tc(q2h, q2l, linv3)  # Q2 D^T (m x kq)
    del q2h, q2l
    check(ops.L.rgsv_axpy(_dev.vp(corr), corr.stride(0), _dev.vp(q2), kp, m, kp, 1.0, ops.st()),
          "axpy")  # Q = Q2 + Q2 D^T
    return corr if kq == kp else corr[:, :kp].contiguous()


def tf32_chain(a: "_dev.DevMatrix", k: int, q: int, seed: int, lo: torch.Tensor | None = None,
               reduce=_noreduce, rows_total: int | None = None):
    """Fixed-rank chain (sketch, shifted CholeskyQR3, q power iterations,
    projection; rangefinder.py:115-123 + SURVEY.md §8(c)) with the four G
    passes on the tf32x3 tensor-core kernels. Returns (Q: m x kp fp64,
    B = Q^T G: kp x ldn fp64, residual history). `lo` may pass a reusable
    (rows x ld) fp32 buffer for G's low part. Row-sharded use (dist.py): `a`
    is this rank's row block, `reduce` all-reduces the k x k Grams, Z^T, B
    and ||G||^2 partials over the ranks and `rows_total` is the global row
    count (CholeskyQR shift)."""
    from .rangefinder import _Ops

    ops = _Ops()
    t = TF32Ops()
    m, n = a.rows, a.cols
    mt = rows_total or m
    if k > min(mt, n):
        raise ValidationError(f"max_cols={k} exceeds min(rows, cols)={min(mt, n)}")
    kp, ldn = _dev.ceil16(k), _dev.ceil16(n)
    kq = _ceil(kp, 32)
    glo, ss = t.split_big(a, lo)
    reduce(ss)
    om = _dev.omega_device(n, k, [seed], ldo=ldn)[0]
    ops.status.zero_()

    def pass_gx(xt):
        xh, xl = t.split_small(xt, kp, ldn, ldn, rows_out=kq)
        y = torch.empty((m, kq), dtype=F64, device="cuda")
        t.gx(a, glo, xh, xl, y, m, kq, n)
        return y if kq == kp else y[:, :kp].contiguous()

    def pass_gtq(qm):
        qh, ql = t.split_small(qm, m, kp, kq)
        out = torch.zeros((kq, ldn), dtype=F64, device="cuda")
        t.gtq(qh, ql, a, glo, out, kq, n, m)
        return reduce(out)[:kp]

    y = pass_gx(om)
    gf2 = float(ss.item())
    if not math.isfinite(gf2):
        raise ValidationError("g contains non-finite entries")
    qm = cholqr_mixed(ops, t, y, m, k, kp, final=q == 0, reduce=reduce, rows_total=mt)
    for it in range(q):
        zt = pass_gtq(qm)
        qht = ops.wide_cholqr3(zt.contiguous(), n, ldn, k, kp)
        y = pass_gx(qht)
        qm = cholqr_mixed(ops, t, y, m, k, kp, final=it == q - 1, reduce=reduce,
                          rows_total=mt)
    b = pass_gtq(qm).contiguous()
    energy = ops.sumsq(_dev.vp(b), ldn, k, n)
    if int(ops.status.item()) & ST_CHOL:
        raise RankDeficiencyError("CholeskyQR breakdown in the range finder (rank-deficient sketch)")
    return qm, b, _dev.residual_history(gf2, energy)
