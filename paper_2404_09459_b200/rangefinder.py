"""Randomized range finder (reference ``rgsv/rangefinder.py``, Alg. 1).

``ExtractionConfig`` keeps every reference field (rangefinder.py:23-49)
and adds ``power_iters`` (q, default 0 = reference behaviour; the
BASELINE configs use q >= 1). ``extract_basis`` runs on
the B200: one fixed-width block (the BASELINE configs' mode) is a single
``rgsv_sketch_project`` call — sketch Y = GΩ, shifted CholeskyQR3,
q power iterations, projection B = QᵀG and its captured energy.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import device as _dev
from ._native import ST_NONFINITE, lib
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


def extract_basis(g, cfg: ExtractionConfig | None = None, *, device_result: bool = False):
    """Extract an approximate orthonormal basis of range(g) on the B200
    (rangefinder.py:68-135). Returns the reference's ``BasisResult``; with
    ``device_result=True`` the basis stays in HBM as a torch tensor."""
    cfg = cfg or ExtractionConfig()
    a = _dev.to_device(g, "g")
    m, n = a.rows, a.cols
    check_max_cols(cfg, m, n)
    width = single_block_width(cfg, m, n)
    if width is None:
        raise ValidationError(
            "the B200 range finder runs the single-block (fixed-rank) mode: set "
            "max_cols <= blocksize (or blocksize >= n) and trim_tol = 0; adaptive multi-block "
            "extraction is not implemented on the device yet")
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
    if code & 0x1:
        raise RankDeficiencyError("CholeskyQR breakdown in the range finder (rank-deficient sketch)")
    if code & ST_NONFINITE:
        raise ValidationError("g contains non-finite entries")
    hist = _dev.residual_history(gf2, energy)
    q = plan.q[:, :width]
    return BasisResult(q if device_result else q.cpu().numpy(), hist, hist[-1] < tol, 1, [width])


def residual_norm(g, q) -> float:
    """Explicit ||(I - QQ^H)G||_F on the device (rangefinder.py:138-154)."""
    a = _dev.to_device(g, "g")
    qa = q if isinstance(q, torch.Tensor) else torch.from_numpy(np.asarray(q, dtype=np.float64))
    if qa.dim() != 2:
        raise DimensionError(f"q must be 2-D, got shape {tuple(qa.shape)}")
    if qa.shape[0] != a.rows:
        raise DimensionError(f"q has {qa.shape[0]} rows but g has {a.rows}")
    if qa.shape[1] == 0:
        return math.sqrt(_dev.device_sumsq(a))
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
    proj = torch.zeros((a.rows, a.ld), dtype=torch.float64, device="cuda")
    # QQ^T G = Q (Q^T G): gx with A = Q (rows x lp), Bt = (Q^T G)^T (cols x lp)
    check(L.rgsv_gemm_gx(_dev.vp(qp), lp, _dev.vp(bt), lp, _dev.vp(proj), a.ld, a.rows, a.cols,
                         lp, _dev.vp(scratch), scratch.numel() * 8, st), "Q (Q^T G)")
    resid = _dev.DevMatrix((a.t - proj[:, : a.cols]).contiguous(), a.rows, a.cols)
    return math.sqrt(_dev.device_sumsq(resid))


__all__ = ["ExtractionConfig", "BasisResult", "extract_basis", "residual_norm"]
