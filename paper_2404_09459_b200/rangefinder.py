"""Randomized range finder (reference ``rgsv/rangefinder.py``, Alg. 1).

``ExtractionConfig`` keeps every reference field (rangefinder.py:23-49)
and adds ``power_iters`` (q, default 0 = reference behaviour; the
BASELINE configs use q >= 1). ``extract_basis`` runs on
the B200: one fixed-width block (the BASELINE configs' mode) is a single
``rgsv_sketch_project`` call — sketch Y = GΩ, shifted CholeskyQR3,
q power iterations, projection B = QᵀG and its captured energy. The
reference's default adaptive mode (several blocks, re-projection against the
growing basis, rank trimming, early stop) runs as a host-driven loop of the
same device kernels (``adaptive_device``), one host sync per block.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import device as _dev
from ._native import ST_CHOL, ST_NONFINITE, check, lib

RGSV_ERR_WORKSPACE = 6  # include/rgsv_b200.h
from .errors import DimensionError, RankDeficiencyError, ValidationError


@dataclass(frozen=True)
class ExtractionConfig:
    """Knobs for basis extraction (rangefinder.py:23-49) + power_iters."""

    tol: float | None = None
    blocksize: int = 100
    seed: int = 0
    max_cols: int | None = None
    trim_tol: float = 1e-12
    power_iters: int = 0

    def __post_init__(self):
        if self.tol is not None and not self.tol > 0:
            raise ValidationError(f"tol must be positive, got {self.tol}")
        if self.blocksize < 1:
            raise ValidationError(f"blocksize must be >= 1, got {self.blocksize}")
        if self.max_cols is not None and self.max_cols < 1:
            raise ValidationError(f"max_cols must be >= 1, got {self.max_cols}")
        if self.trim_tol < 0:
            raise ValidationError(f"trim_tol must be >= 0, got {self.trim_tol}")
        if self.power_iters < 0:
            raise ValidationError(f"power_iters must be >= 0, got {self.power_iters}")

    @staticmethod
    def fixed_rank(k: int, seed: int = 0, power_iters: int = 0) -> "ExtractionConfig":
        """One block of exactly k columns, no trimming, no early stop — the
        form the reference's own tests use for a fixed-width sketch
        (test_bounds.py:71-74)."""
        return ExtractionConfig(tol=1e-300, blocksize=k, seed=seed, max_cols=k, trim_tol=0.0,
                                power_iters=power_iters)


@dataclass
class BasisResult:
    """Output of ``extract_basis`` (rangefinder.py:52-65)."""

    q: np.ndarray
    residual_history: list
    converged: bool
    iterations: int
    block_widths: list = field(default_factory=list)


def single_block_width(cfg: ExtractionConfig, m: int, n: int) -> int | None:
    """Width of the one block the reference loop would run when the loop is
    guaranteed to stop after its first block (rangefinder.py:104-133):
    either there is only one block or the first block reaches max_cols,
    and no column can be trimmed (trim_tol == 0). None otherwise."""
    b = min(cfg.blocksize, n)
    width = b
    if cfg.max_cols is not None:
        width = min(width, cfg.max_cols)
    one_block = (-(-n // b) == 1) or (cfg.max_cols is not None and width >= cfg.max_cols)
    if one_block and cfg.trim_tol == 0.0:
        return width
    return None


def check_max_cols(cfg: ExtractionConfig, m: int, n: int) -> None:
    if cfg.max_cols is not None and cfg.max_cols > min(m, n):
        raise ValidationError(f"max_cols={cfg.max_cols} exceeds min(rows, cols)={min(m, n)}")


class _Ops:
    """The device kernels the adaptive loop strings together (C-ABI calls on
    the current stream; scratch and status owned here)."""

    def __init__(self):
        self.L = lib()
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.scratch = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")

    def st(self):
        return _dev.sp(torch.cuda.current_stream())

    def _scr(self, need: int):
        if self.scratch.numel() < need:
            self.scratch = torch.empty(need, dtype=torch.uint8, device="cuda")

    def _gemm(self, fn, name, *args):
        # split-K partials need scratch that depends on the tile plan: grow
        # on RGSV_ERR_WORKSPACE (checked before any launch) and retry
        while True:
            rc = fn(*args, _dev.vp(self.scratch), self.scratch.numel(), self.st())
            if rc != RGSV_ERR_WORKSPACE:
                return check(rc, name)
            self._scr(self.scratch.numel() * 4)

    def gx(self, a, lda, bt, ldb, out, ldc, M, N, K):
        """out (M x N) = A (M x K) Bt^T."""
        self._gemm(self.L.rgsv_gemm_gx, "gemm_gx", a, lda, bt, ldb, out, ldc, M, N, K)

    def gtq(self, a, lda, b, ldb, out, ldc, M, N, K):
        """out (M x N) = A^T B with A: K x M, B: K x N."""
        self._gemm(self.L.rgsv_gemm_gtq, "gemm_gtq", a, lda, b, ldb, out, ldc, M, N, K)

    def gram(self, a, lda, kp, rows, out):
        """out (kp x kp) = A^T A: the lower triangle, on the tiles that touch
        it (rgsv_gemm_gram_lower) when kp > 128 (the blocked Cholesky reads
        only the lower part); the full product otherwise."""
        if kp > 128:
            self._gemm(self.L.rgsv_gemm_gram_lower, "gemm_gram_lower", a, lda, kp, rows, out, kp)
        else:
            self.gtq(a, lda, a, lda, out, kp, kp, kp, rows)

    def chol(self, gram, k, kp, shift_rows):
        linv = torch.zeros(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
        rinv = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
        rdiag = torch.zeros(kp, dtype=torch.float64, device="cuda")
        check(self.L.rgsv_chol_inv(_dev.vp(gram), k, kp, shift_rows, _dev.vp(linv),
                                   _dev.vp(rinv), _dev.vp(rdiag), _dev.vp(self.status),
                                   self.st()), "chol_inv")
        return linv[: kp * kp].view(kp, kp), rinv

    def cholqr3(self, y, m, k, kp):
        """Shifted CholeskyQR3 of y (m x kp, columns >= k zero): Q (m x kp)."""
        for step in range(3):
            gram = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
            self.gtq(_dev.vp(y), kp, _dev.vp(y), kp, _dev.vp(gram), kp, kp, kp, m)
            linv, _ = self.chol(gram, k, kp, m if step == 0 else 0)
            q = torch.zeros((m, kp), dtype=torch.float64, device="cuda")
            self.gx(_dev.vp(y), kp, _dev.vp(linv), kp, _dev.vp(q), kp, m, kp, kp)
            y = q
        return y

    def wide_cholqr3(self, zt, n, ldn, k, kp):
        """Q of qr(Z) for Z = zt^T (zt: kp x ldn): returns Qhat^T (kp x ldn)."""
        src = zt
        for step in range(3):
            gram = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
            self.gx(_dev.vp(src), ldn, _dev.vp(src), ldn, _dev.vp(gram), kp, kp, kp, n)
            _, rinv = self.chol(gram, k, kp, n if step == 0 else 0)
            dst = torch.zeros((kp, ldn), dtype=torch.float64, device="cuda")
            self.gtq(_dev.vp(rinv), kp, _dev.vp(src), ldn, _dev.vp(dst), ldn, kp, n, kp)
            src = dst
        return src

    def householder(self, y, m, w, kp):
        """Robust QR (rgsv_householder_qr): Q (m x kp, zero-padded), |diag R|."""
        a = y.clone()
        q = torch.zeros((m, kp), dtype=torch.float64, device="cuda")
        rd = torch.zeros(kp, dtype=torch.float64, device="cuda")
        tau = torch.zeros(kp, dtype=torch.float64, device="cuda")
        check(self.L.rgsv_householder_qr(_dev.vp(a), kp, m, w, _dev.vp(q), kp, _dev.vp(rd),
                                         _dev.vp(tau), self.st()), "householder_qr")
        return q, rd[: min(m, w)]

    def reproject(self, y, m, wp, q, lqp):
        """y -= Q (Q^T y), twice (rangefinder.py:116-118)."""
        for _ in range(2):
            tt = torch.zeros((wp, lqp), dtype=torch.float64, device="cuda")
            self.gtq(_dev.vp(y), wp, _dev.vp(q), q.stride(0), _dev.vp(tt), lqp, wp, lqp, m)
            proj = torch.zeros((m, wp), dtype=torch.float64, device="cuda")
            self.gx(_dev.vp(q), q.stride(0), _dev.vp(tt), lqp, _dev.vp(proj), wp, m, wp, lqp)
            check(self.L.rgsv_axpy(_dev.vp(y), wp, _dev.vp(proj), wp, m, wp, -1.0, self.st()),
                  "axpy")

    def sumsq(self, a, lda, rows, cols) -> float:
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        ws = torch.zeros(1024, dtype=torch.float64, device="cuda")
        check(self.L.rgsv_sumsq(a, lda, rows, cols, _dev.vp(out), _dev.vp(ws), 8192,
                                self.st()), "sumsq")
        return float(out.item())


# smallest |R_jj| / max |R_jj| a block may have and still take CholeskyQR3
# (RGSV_CHOLQR_COND overrides; the one-CTA Householder fallback is ~100x slower)
RGSV_CHOLQR_COND = float(os.environ.get("RGSV_CHOLQR_COND", "1e-13"))


def _block_qr(ops: _Ops, y, m: int, w: int, wp: int, trim_cut: float):
    """reduced_qr of one sketch block with the reference's phase (core.py:80-95)
    and |diag R| for the trim test. Well-conditioned blocks take shifted
    CholeskyQR3 (R_jj = q_j^T y_j from one small GEMM); blocks whose R is
    near the trim threshold or numerically rank deficient -- where the trim
    decision needs Householder's rank-revealing diagonal -- take the robust
    one-CTA Householder kernel."""
    mode = os.environ.get("RGSV_ADAPTIVE_QR", "auto")  # diagnostics: auto|householder
    if m >= w and mode != "householder":
        ops.status.zero_()
        q = ops.cholqr3(y, m, w, wp)
        r = torch.zeros((wp, wp), dtype=torch.float64, device="cuda")
        ops.gtq(_dev.vp(q), wp, _dev.vp(y), wp, _dev.vp(r), wp, wp, wp, m)
        rd = torch.diagonal(r)[:w].abs().cpu().numpy()
        ok = (int(ops.status.item()) & (ST_CHOL | ST_NONFINITE)) == 0
        # shifted CholeskyQR3 is backward stable up to cond ~ 1/u (Fukaya et
        # al. 2020), so only blocks near the trim threshold or beyond that
        # conditioning need Householder's rank-revealing diagonal
        # the trim decision (|R_jj| >= trim_cut) must match Householder's: the
        # CholeskyQR diagonal agrees with it to ~cond * u relative, so a block
        # whose smallest |R_jj| clears the cut by a condition-scaled margin
        # (1e-10 * max/min, i.e. >= 1e6 u * cond) decides the same way
        if ok and np.all(np.isfinite(rd)) and rd.min() > 0.0:
            margin = 1.0 + 1e-10 * rd.max() / rd.min()
            if rd.min() >= max(margin * trim_cut, RGSV_CHOLQR_COND * rd.max()):
                return q, rd
    q, rd = ops.householder(y, m, w, wp)
    return q, rd.cpu().numpy()


def adaptive_device(a: "_dev.DevMatrix", cfg: ExtractionConfig):
    """Alg. 1 (rangefinder.py:68-135) on the device. Returns
    (Q: m x lq tensor, B = Q^T G: lq x ldn tensor, BasisResult). Block i's
    Omega continues the ONE generator stream (offset = normals drawn so far),
    so every block is bit-identical to the reference's draw."""
    ops = _Ops()
    m, n = a.rows, a.cols
    ldn = _dev.ceil16(n)
    gf2 = _dev.device_sumsq(a)                                   # :83
    if not math.isfinite(gf2):
        raise ValidationError("g contains non-finite entries")
    normf = math.sqrt(gf2)
    tol = cfg.tol if cfg.tol is not None else 1e-10 * normf      # :85
    trim_cut = cfg.trim_tol * normf                              # :86
    # every sampled column may be kept (trim_tol = 0 keeps noise columns too,
    # rangefinder.py:120-124), so the basis can hold up to n (or max_cols)
    cap = n if cfg.max_cols is None else cfg.max_cols
    capp = _dev.ceil16(cap)
    qb = torch.zeros((m, capp), dtype=torch.float64, device="cuda")
    bb = torch.zeros((capp, ldn), dtype=torch.float64, device="cuda")
    history = [normf]
    widths: list = []
    lq = 0
    if normf == 0.0 or normf < tol:                              # :96
        return qb[:, :0], bb[:0], BasisResult(None, history, True, 0, widths)
    b = min(cfg.blocksize, n)                                    # :99
    nblocks = -(-n // b)
    captured: list = []
    converged = False
    iterations = 0
    offset = 0
    for i in range(nblocks):                                     # :106
        width = min(b, n - i * b)
        if cfg.max_cols is not None:
            width = min(width, cfg.max_cols - lq)
            if width <= 0:
                break
        wp = _dev.ceil16(width)
        om = _dev.omega_block(n, width, cfg.seed, offset, ldn)    # :112
        offset += n * width
        y = torch.zeros((m, wp), dtype=torch.float64, device="cuda")
        ops.gx(_dev.vp(a.t), a.ld, _dev.vp(om), ldn, _dev.vp(y), wp, m, wp, n)  # :115
        lqp = _dev.ceil16(lq)
        if lq:
            ops.reproject(y, m, wp, qb, lqp)                     # :116-118
        for _ in range(cfg.power_iters):
            p, _ = _block_qr(ops, y, m, width, wp, 0.0)
            zt = torch.zeros((wp, ldn), dtype=torch.float64, device="cuda")
            ops.gtq(_dev.vp(p), wp, _dev.vp(a.t), a.ld, _dev.vp(zt), ldn, wp, n, m)
            qht = ops.wide_cholqr3(zt, n, ldn, width, wp)
            y = torch.zeros((m, wp), dtype=torch.float64, device="cuda")
            ops.gx(_dev.vp(a.t), a.ld, _dev.vp(qht), ldn, _dev.vp(y), wp, m, wp, n)
            if lq:
                ops.reproject(y, m, wp, qb, lqp)
        p, rd = _block_qr(ops, y, m, width, wp, trim_cut)        # :119
        keep = np.flatnonzero(rd >= trim_cut)                    # :120-121
        kc = int(keep.size)
        if kc:
            pk = torch.zeros((m, wp), dtype=torch.float64, device="cuda")
            if kc == width:
                pk.copy_(p)
            else:
                pk[:, :kc] = p[:, torch.from_numpy(keep).cuda()]
            blk = torch.zeros((wp, ldn), dtype=torch.float64, device="cuda")
            ops.gtq(_dev.vp(pk), wp, _dev.vp(a.t), a.ld, _dev.vp(blk), ldn, wp, n, m)
            captured.append(ops.sumsq(_dev.vp(blk), ldn, kc, n))  # :123
            qb[:, lq: lq + kc] = pk[:, :kc]                      # :124
            bb[lq: lq + kc] = blk[:kc]
            lq += kc
        widths.append(kc)
        res2 = gf2 - math.fsum(captured)                         # :126
        history.append(math.sqrt(max(res2, 0.0)))
        iterations = i + 1
        if history[-1] < tol:                                    # :129-131
            converged = True
            break
        if cfg.max_cols is not None and lq >= cfg.max_cols:      # :132-133
            break
    return qb[:, :lq], bb[:lq], BasisResult(None, history, converged, iterations, widths)


def chunked_chain(a: "_dev.DevMatrix", k: int, q: int, seed: int, chunk_rows: int | None = None):
    """The fixed-rank chain (sketch, shifted CholeskyQR3, q power iterations,
    projection: rangefinder.py:115-123 + SURVEY.md §8(c)) with G streamed in
    fp64 row chunks -- fp32 input is promoted chunk by chunk (the reference
    promotes up front, core.py:51-54). Every GEMM pass converts each chunk
    once and runs the DMMA GEMM on it; the Q^T G partials of the chunks are
    summed in chunk order. Returns (Q: m x kp, B = Q^T G: kp x ldn, residual
    history)."""
    ops = _Ops()
    m, n = a.rows, a.cols
    if k > min(m, n):
        raise ValidationError(f"max_cols={k} exceeds min(rows, cols)={min(m, n)}")
    kp, ldn = _dev.ceil16(k), _dev.ceil16(n)
    f64 = torch.float64
    om = _dev.omega_device(n, k, [seed], ldo=ldn)[0]
    ops.status.zero_()

    def chunks():
        return _dev.f64_chunks(a, chunk_rows)

    def pass_gx(xt):
        y = torch.zeros((m, kp), dtype=f64, device="cuda")
        ss = []
        for r0, r1, c in chunks():
            ops.gx(_dev.vp(c.t), c.ld, _dev.vp(xt), ldn, _dev.vp(y[r0:]), kp, r1 - r0, kp, n)
            if xt is om:
                ss.append(ops.sumsq(_dev.vp(c.t), c.ld, r1 - r0, n))
        return y, ss

    def pass_gtq(qm):
        acc = torch.zeros((kp, ldn), dtype=f64, device="cuda")
        part = torch.zeros((kp, ldn), dtype=f64, device="cuda") if a.is_f32 else acc
        for r0, r1, c in chunks():
            ops.gtq(_dev.vp(qm[r0:]), kp, _dev.vp(c.t), c.ld, _dev.vp(part), ldn, kp, n, r1 - r0)
            if part is not acc:
                check(ops.L.rgsv_axpy(_dev.vp(acc), ldn, _dev.vp(part), ldn, kp, ldn, 1.0,
                                      ops.st()), "axpy")
        return acc

    y, ss = pass_gx(om)
    gf2 = math.fsum(ss)
    if not math.isfinite(gf2):
        raise ValidationError("g contains non-finite entries")
    qm = ops.cholqr3(y, m, k, kp)
    for _ in range(q):
        zt = pass_gtq(qm)
        qht = ops.wide_cholqr3(zt, n, ldn, k, kp)
        y, _ = pass_gx(qht)
        qm = ops.cholqr3(y, m, k, kp)
    b = pass_gtq(qm)
    energy = ops.sumsq(_dev.vp(b), ldn, k, n)
    if int(ops.status.item()) & ST_CHOL:
        raise RankDeficiencyError("CholeskyQR breakdown in the range finder (rank-deficient sketch)")
    return qm, b, _dev.residual_history(gf2, energy)


def extract_basis(g, cfg: ExtractionConfig | None = None, *, device_result: bool = False):
    """Extract an approximate orthonormal basis of range(g) on the B200
    (rangefinder.py:68-135). Returns the reference's ``BasisResult``; with
    ``device_result=True`` the basis stays in HBM as a torch tensor. A
    fixed-width single block takes the fused ``rgsv_sketch_project`` call;
    any other configuration runs ``adaptive_device``."""
    cfg = cfg or ExtractionConfig()
    a = _dev.to_device(g, "g")
    m, n = a.rows, a.cols
    check_max_cols(cfg, m, n)
    width = single_block_width(cfg, m, n)
    if width is None:
        q, _, res = adaptive_device(a, cfg)
        res.q = q if device_result else q.cpu().numpy()
        return res
    if width > 128:  # beyond the fused call's sketch (N <= 128): separate launches
        gf2 = _dev.device_sumsq(a)
        if not math.isfinite(gf2):
            raise ValidationError("g contains non-finite entries")
        normf = math.sqrt(gf2)
        tol = cfg.tol if cfg.tol is not None else 1e-10 * normf
        if normf == 0.0 or normf < tol:  # rangefinder.py:96
            q0 = torch.zeros((m, 0), dtype=torch.float64, device="cuda")
            return BasisResult(q0 if device_result else q0.cpu().numpy(), [normf], True, 0, [])
        q, _, hist = chunked_chain(a, width, cfg.power_iters, cfg.seed)
        q = q[:, :width]
        return BasisResult(q if device_result else q.cpu().numpy(), hist, hist[-1] < tol, 1,
                           [width])
    plan = _dev.SketchPlan(m, n, width)
    stats = torch.zeros(2, dtype=torch.float64, device="cuda")
    rdiag = torch.zeros(max(width, 1), dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    plan.set_seed(cfg.seed)
    plan.enqueue_omega(status, st)
    plan.launch(a, cfg.power_iters, stats, rdiag, status, st)
    gf2, energy = (float(x) for x in stats.cpu().tolist())
    code = int(status.item())
    if not math.isfinite(gf2):
        raise ValidationError("g contains non-finite entries")
    normf = math.sqrt(gf2)
    tol = cfg.tol if cfg.tol is not None else 1e-10 * normf
    if normf == 0.0 or normf < tol:  # rangefinder.py:96: no sampling at all
        q0 = torch.zeros((m, 0), dtype=torch.float64, device="cuda")
        return BasisResult(q0 if device_result else q0.cpu().numpy(), [normf], True, 0, [])
    if code & ST_NONFINITE:
        raise ValidationError("g contains non-finite entries")
    if code & 0x1:
        # the sketch is wider than the numerical rank of g (exactly low-rank
        # input): CholeskyQR breaks down where the reference's Householder QR
        # keeps the columns (rangefinder.py:119-124, trim_tol = 0); the general
        # loop factors such a block with the Householder kernel
        q, _, res = adaptive_device(a, cfg)
        res.q = q if device_result else q.cpu().numpy()
        return res
    hist = _dev.residual_history(gf2, energy)
    q = plan.q[:, :width]
    return BasisResult(q if device_result else q.cpu().numpy(), hist, hist[-1] < tol, 1, [width])


def projected(a: "_dev.DevMatrix", q) -> torch.Tensor:
    """Q (Q^T G) on the device (two DMMA GEMMs): the rows x cols projection
    of G onto the basis' range, as residual_norm (rangefinder.py:138-154)
    and the CLI's bounds command (cli.py:164-165) form it."""
    qa = q if isinstance(q, torch.Tensor) else torch.from_numpy(np.asarray(q, dtype=np.float64))
    if qa.dim() != 2:
        raise DimensionError(f"q must be 2-D, got shape {tuple(qa.shape)}")
    if qa.shape[0] != a.rows:
        raise DimensionError(f"q has {qa.shape[0]} rows but g has {a.rows}")
    proj = torch.zeros((a.rows, a.cols + (a.cols & 1)), dtype=torch.float64, device="cuda")
    if qa.shape[1] == 0:
        return proj[:, : a.cols]
    L = lib()
    qd = qa.to("cuda", torch.float64)
    l = qd.shape[1]
    lp = _dev.ceil16(l)
    qp = torch.zeros((a.rows, lp), dtype=torch.float64, device="cuda")
    qp[:, :l] = qd
    ldb = _dev.ceil16(a.cols)
    b = torch.zeros((lp, ldb), dtype=torch.float64, device="cuda")
    scratch = torch.empty(148 * lp * ldb + 4096, dtype=torch.float64, device="cuda")
    st = _dev.sp(torch.cuda.current_stream())
    from ._native import check

    check(L.rgsv_gemm_gtq(_dev.vp(qp), lp, _dev.vp(a.t), a.ld, _dev.vp(b), ldb, lp, a.cols,
                          a.rows, _dev.vp(scratch), scratch.numel() * 8, st), "Q^T G")
    bt = torch.zeros((a.cols + (a.cols & 1), lp), dtype=torch.float64, device="cuda")
    bt[: a.cols, :] = b[:, : a.cols].t()
    # QQ^T G = Q (Q^T G): gx with A = Q (rows x lp), Bt = (Q^T G)^T (cols x lp)
    check(L.rgsv_gemm_gx(_dev.vp(qp), lp, _dev.vp(bt), lp, _dev.vp(proj), proj.stride(0), a.rows,
                         a.cols, lp, _dev.vp(scratch), scratch.numel() * 8, st), "Q (Q^T G)")
    return proj[:, : a.cols]


def residual_norm(g, q) -> float:
    """Explicit ||(I - QQ^H)G||_F on the device (rangefinder.py:138-154)."""
    a = _dev.to_device(g, "g")
    proj = projected(a, q)
    resid = _dev.DevMatrix((a.t - proj).contiguous(), a.rows, a.cols)
    return math.sqrt(_dev.device_sumsq(resid))


__all__ = ["ExtractionConfig", "BasisResult", "extract_basis", "residual_norm"]
