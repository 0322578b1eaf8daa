"""Generalized singular values of a matrix pair (reference ``rgsv/engine.py``).

``compute_gsv`` / ``compare`` run the whole randomized pipeline on the B200
(device.PairPlan): both range-finder chains, the stacked QR + Jacobi SVD of
the L blocks and the fused spectrum/comparative kernel, with one packed
device->host copy at the end. The result types, their invariants and the
error behaviour follow the reference line by line (citations inline).
"""

from __future__ import annotations

import dataclasses
import math
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np
import torch

from . import device as _dev
from . import tf32 as _tf32
from ._native import (ST_CHOL, ST_CLASSIFY, ST_JACOBI, ST_NONFINITE, ST_OMEGA_SHORT,
                      ST_SPECTRUM)
from ._native import check as _check
from ._native import lib as _native_lib
from .errors import (
    ConvergenceError,
    DimensionError,
    RankDeficiencyError,
    RecoveryError,
    ValidationError,
)
from .rangefinder import (
    BasisResult,
    ExtractionConfig,
    adaptive_device,
    chunked_chain,
    check_max_cols,
    single_block_width,
)

RANDOMIZED = "randomized"
DIRECT = "direct"


@dataclass(frozen=True)
class GmpPair:
    """A pair {g1 (m x n), g2 (p x n)} held in HBM (engine.py:31-90).

    Construction validates shapes, the field (real only on the B200 path),
    finiteness (device pass) and m + p >= n, and -- like the reference --
    sigma_min > 1e-12 sigma_max of the stacked pair (engine.py:55-61), on the
    device (validation.py: Householder or CholeskyQR3 R factor, then blocked
    Jacobi). ``check_rank=None`` (default) and True both run the check; it
    covers n <= 4096 (every reference shape and cfg0-cfg3) and raises
    DimensionError beyond (cfg4: n = 8192), where the pair must be built
    with check_rank=False. With False the stacked norms (stack_norm2,
    stack_pinv_norm) are computed on first access instead."""

    g1: object
    g2: object
    check_rank: bool | None = None

    def __post_init__(self):
        a = _dev.to_device(self.g1, "g1", keep_f32=True)
        b = _dev.to_device(self.g2, "g2", keep_f32=True)
        if a.cols != b.cols:
            raise DimensionError(f"g1 has {a.cols} columns but g2 has {b.cols}")
        n = a.cols
        if a.rows + b.rows < n:
            raise RankDeficiencyError(f"stacked pair has {a.rows + b.rows} rows < {n} columns")
        for name, g in (("g1", a), ("g2", b)):
            if not math.isfinite(_dev.device_sumsq(g)):
                raise ValidationError(f"{name} contains non-finite entries")
        object.__setattr__(self, "g1", a)
        object.__setattr__(self, "g2", b)
        if self.check_rank is not False:
            self._stack_norms()

    def _stack_norms(self):
        """sigma_max / sigma_min of vstack(g1, g2) (engine.py:55-61, 82-90),
        computed once on the device; RankDeficiencyError like the reference."""
        if not hasattr(self, "_stack_smax"):
            from .validation import stacked_extreme_singular_values

            smax, smin = stacked_extreme_singular_values(self.g1, self.g2)
            if smin <= 1e-12 * smax:
                raise RankDeficiencyError(
                    f"stacked pair is numerically rank deficient "
                    f"(sigma_min/sigma_max = {smin / smax if smax else 0.0:.3e})")
            object.__setattr__(self, "_stack_smax", smax)
            object.__setattr__(self, "_stack_smin", smin)
        return self._stack_smax, self._stack_smin

    @classmethod
    def resident(cls, g1, g2) -> "GmpPair":
        """Wrap device matrices without the validation passes (the bench
        path: G already resident in HBM, validated once at creation)."""
        pair = object.__new__(cls)
        object.__setattr__(pair, "g1", _dev.to_device(g1, "g1", keep_f32=True))
        object.__setattr__(pair, "g2", _dev.to_device(g2, "g2", keep_f32=True))
        object.__setattr__(pair, "check_rank", False)
        return pair

    @property
    def m(self) -> int:
        return self.g1.rows

    @property
    def p(self) -> int:
        return self.g2.rows

    @property
    def n(self) -> int:
        return self.g1.cols

    def stacked(self) -> np.ndarray:
        return np.vstack([self.g1.t.cpu().numpy(), self.g2.t.cpu().numpy()])

    @property
    def stack_norm2(self) -> float:
        """Largest singular value of the stacked pair (cached; engine.py:82-85)."""
        return self._stack_norms()[0]

    @property
    def stack_pinv_norm(self) -> float:
        """Spectral norm of the stacked pair's pseudoinverse (engine.py:87-90)."""
        return 1.0 / self._stack_norms()[1]


@dataclass(frozen=True)
class GsvSpectrum:
    """Paired GSV sequences with block counts (engine.py:93-129); the
    invariants are checked exactly as the reference does."""

    alphas: np.ndarray
    betas: np.ndarray
    r: int
    s: int

    def __post_init__(self):
        a = np.asarray(self.alphas, dtype=np.float64)
        b = np.asarray(self.betas, dtype=np.float64)
        if a.ndim != 1 or b.ndim != 1 or a.size != b.size or a.size == 0:
            raise DimensionError("alphas and betas must be 1-D of equal, nonzero length")
        n = a.size
        if self.r < 0 or self.s < 0 or self.r + self.s > n:
            raise ValidationError(f"invalid counts r={self.r}, s={self.s} for n={n}")
        if np.any(a < 0) or np.any(a > 1) or np.any(b < 0) or np.any(b > 1):
            raise ValidationError("GSVs must lie in [0, 1]")
        if np.any(np.diff(a) > 1e-12) or np.any(np.diff(b) < -1e-12):
            raise ValidationError("alphas must be nonincreasing and betas nondecreasing")
        if float(np.max(np.abs(a**2 + b**2 - 1.0))) > 1e-12:
            raise ValidationError("alpha_i^2 + beta_i^2 = 1 violated beyond 1e-12")
        if np.any(b[: self.r] != 0.0) or np.any(a[self.r + self.s:] != 0.0):
            raise ValidationError("classified-zero entries must be exactly 0")
        object.__setattr__(self, "alphas", a)
        object.__setattr__(self, "betas", b)

    @property
    def n(self) -> int:
        return self.alphas.size


@dataclass(frozen=True)
class GsvOptions:
    """Method selection and thresholds (engine.py:132-150)."""

    extraction: ExtractionConfig = ExtractionConfig()
    classify_tol: float = 1e-10
    method: str = RANDOMIZED
    # fp32-resident pairs (not in the reference, which promotes fp32 to fp64
    # up front, core.py:51-54): "tf32x3" runs the G passes on the tcgen05
    # tensor cores at fp32-level accuracy (tf32.py); "promote" streams
    # fp64-promoted row chunks through the DMMA chain (the reference's exact
    # arithmetic).
    f32_mode: str = "tf32x3"

    def __post_init__(self):
        if self.f32_mode not in ("tf32x3", "promote"):
            raise ValidationError(f"f32_mode must be 'tf32x3' or 'promote', got {self.f32_mode!r}")
        if not 0 < self.classify_tol < 1e-2:
            raise ValidationError(f"classify_tol must be in (0, 1e-2), got {self.classify_tol}")
        if self.method not in (RANDOMIZED, DIRECT):
            raise ValidationError(
                f"method must be 'randomized' or 'direct', got {self.method!r}")


@dataclass(frozen=True)
class GsvdFactors:
    """G1 = U diag(alpha) R, G2 = V diag(beta) R (engine.py:153-161)."""

    u: np.ndarray
    v: np.ndarray
    r_factor: np.ndarray
    spectrum: GsvSpectrum


def classify_spectrum(alphas, betas, classify_tol: float = 1e-10) -> tuple[int, int]:
    """(r, s) block counts with in-place snapping (engine.py:164-186).
    Operates on caller-owned arrays, as the reference does; the device
    pipeline performs the same classification inside its fused kernel."""
    if not 0 < classify_tol < 1e-2:
        raise ValidationError(f"classify_tol must be in (0, 1e-2), got {classify_tol}")
    a = np.asarray(alphas)
    b = np.asarray(betas)
    n = a.size
    r = int(np.count_nonzero(b < classify_tol))
    za = int(np.count_nonzero(a < classify_tol))
    s = n - r - za
    if s < 0:
        raise ValidationError("overlapping zero classifications; sequences not ordered?")
    b[:r] = 0.0
    a[:r] = 1.0
    if za:
        a[n - za:] = 0.0
        b[n - za:] = 1.0
    return r, s


def spectrum_from_l_blocks(l1_block, l2_block, n: int, classify_tol: float = 1e-10,
                           branch: str | None = None) -> GsvSpectrum:
    """GSVs read off the stacked-QR orthonormal blocks (engine.py:189-225)
    on the device: one-sided Jacobi singular values of both blocks, clamp to
    [0, 1], the merged completion (each index keeps its smaller member and
    completes the other through sqrt(1 - x^2)) or the forced one-sided
    ``branch`` ("first" / "second"), then classify_spectrum's counts and
    snapping (engine.py:164-186) -- rgsv_spectrum_from_l_blocks, one call."""
    if branch not in (None, "first", "second"):
        raise ValidationError(f"branch must be None, 'first' or 'second', got {branch!r}")
    if not 0 < classify_tol < 1e-2:
        raise ValidationError(f"classify_tol must be in (0, 1e-2), got {classify_tol}")
    blocks = []
    for name, blk in (("l1_block", l1_block), ("l2_block", l2_block)):
        if isinstance(blk, torch.Tensor):
            t = blk.to(device="cuda", dtype=torch.float64)
        else:
            t = torch.from_numpy(np.ascontiguousarray(np.asarray(blk, dtype=np.float64))).cuda()
        if t.dim() != 2:
            raise DimensionError(f"{name} must be 2-D")
        blocks.append(t.contiguous())
    b1, b2 = blocks
    l1, c1 = b1.shape
    l2, c2 = b2.shape
    if l1 and l2 and c1 != c2:
        raise DimensionError(f"L blocks have {c1} and {c2} columns")
    cols = c1 if l1 else c2
    L = _native_lib()
    nb = int(L.rgsv_spectrum_from_l_blocks_workspace_bytes(l1, l2, cols, n))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    alphas = torch.empty(n, dtype=torch.float64, device="cuda")
    betas = torch.empty(n, dtype=torch.float64, device="cuda")
    ints = torch.zeros(3, dtype=torch.int32, device="cuda")
    dummy = torch.zeros(1, dtype=torch.float64, device="cuda")
    _check(L.rgsv_spectrum_from_l_blocks(
        _dev.vp(b1 if l1 else dummy), max(c1, 1), l1, _dev.vp(b2 if l2 else dummy), max(c2, 1), l2,
        cols, n, classify_tol, {None: 0, "first": 1, "second": 2}[branch], _dev.vp(alphas),
        _dev.vp(betas), _dev.vp(ints[:2]), _dev.vp(ints[2:]), _dev.vp(ws), nb,
        _dev.sp(torch.cuda.current_stream())), "rgsv_spectrum_from_l_blocks")
    r, s, status = (int(x) for x in ints.cpu())
    if status & ST_JACOBI:
        raise ConvergenceError("Jacobi SVD of an L block did not converge")
    if status & ST_CLASSIFY:
        raise ValidationError("overlapping zero classifications; sequences not ordered?")
    return GsvSpectrum(alphas.cpu().numpy(), betas.cpu().numpy(), r, s)


@dataclass(frozen=True)
class _Pipeline:
    """The reference's internal pipeline record (engine.py:234-242): bases
    (None for method="direct"), the stacked-QR L blocks, R-tilde and the
    BasisResults. Host arrays, as the reference returns them."""

    q1: np.ndarray | None
    q2: np.ndarray | None
    l1_block: np.ndarray
    l2_block: np.ndarray
    r_tilde: np.ndarray
    basis1: object | None = None
    basis2: object | None = None


def _run_pipeline(pair: GmpPair, opts: GsvOptions) -> _Pipeline:
    """engine._run_pipeline (engine.py:245-261) on the device -- the seam the
    reference's bench._timed_run (bench.py:74) and cli._cmd_bounds
    (cli.py:163) call: bases (extract_basis on the device, G2 with seed + 1),
    C_i = Q_i^T G_i (DMMA), the stacked reduced QR [C1; C2] = Q R-tilde
    (multi-CTA Householder for <= 1408 stacked rows, CholeskyQR3 above) with
    the reference's phase convention, L blocks = row blocks of Q."""
    from .core import HH_MAX_ROWS, _gemm_at_b, dense_qr, tall_qr

    if pair.g1.is_f32 or pair.g2.is_f32:
        pair = _promoted(pair)
    n = pair.n
    if opts.method == DIRECT:
        c1, c2 = pair.g1.t, pair.g2.t
        q1 = q2 = None
        b1 = b2 = None
    else:
        from .rangefinder import extract_basis

        cfg = opts.extraction
        b1 = extract_basis(pair.g1, cfg)
        b2 = extract_basis(pair.g2, dataclasses.replace(cfg, seed=cfg.seed + 1))
        q1, q2 = b1.q, b2.q
        cs = []
        for q, g in ((q1, pair.g1), (q2, pair.g2)):
            w = q.shape[1]
            if w == 0:
                cs.append(torch.zeros((0, n), dtype=torch.float64, device="cuda"))
                continue
            qd = torch.zeros((g.rows, _dev.ceil16(w)), dtype=torch.float64, device="cuda")
            qd[:, :w] = torch.from_numpy(np.ascontiguousarray(q)).cuda()
            cs.append(_gemm_at_b(qd, g.t, w, n, g.rows))
        c1, c2 = cs
    l1, l2 = c1.shape[0], c2.shape[0]
    l = l1 + l2
    if l == 0:
        raise RankDeficiencyError("both compressed blocks are empty")
    if l <= HH_MAX_ROWS:
        if l1 and l2:
            q, r = dense_qr(c1, l1, c2, l2, n)
        else:
            q, r = dense_qr(c1 if l1 else c2, l, None, 0, n)
    elif l >= n:
        s_ = torch.zeros((l, n + (n & 1)), dtype=torch.float64, device="cuda")
        s_[:l1, :n] = c1
        s_[l1:, :n] = c2
        q, r = tall_qr(s_[:, :n], l, n)
    else:
        raise DimensionError(f"stacked reduced QR of a wide {l} x {n} block with more than "
                             f"{HH_MAX_ROWS} rows is not supported")
    qh = q.cpu().numpy()
    return _Pipeline(q1, q2, qh[:l1], qh[l1:], r.cpu().numpy(), b1, b2)


@dataclass
class DeviceRun:
    """Everything one device pipeline run produced (host copies of the
    small outputs; bases and projections stay in HBM)."""

    spectrum: GsvSpectrum | None
    alphas: np.ndarray
    betas: np.ndarray
    r: int
    s: int
    rho: np.ndarray
    theta: np.ndarray
    p1: np.ndarray
    p2: np.ndarray
    d1: float
    d2: float
    psum: tuple
    status: int
    basis1: BasisResult
    basis2: BasisResult
    sv1: np.ndarray
    sv2: np.ndarray
    plan: object


def _fixed_width(opts: GsvOptions, m: int, p: int, n: int):
    """(k1, k2) when both chains are one fixed-width block (the fused,
    graph-captured pair pipeline), else None (direct or adaptive mode)."""
    if opts.method == DIRECT:  # no extraction at all (engine.py:246-249)
        return None
    cfg = opts.extraction
    check_max_cols(cfg, m, n)
    check_max_cols(cfg, p, n)
    w1 = single_block_width(cfg, m, n)
    w2 = single_block_width(cfg, p, n)
    if w1 is None or w2 is None:
        return None
    return w1, w2


def _small_checked(c1, l1: int, c2, l2: int, n: int, classify_tol: float) -> dict:
    """device.small_spectrum + the reference's error mapping."""
    out = _dev.small_spectrum(c1, l1, c2, l2, n, classify_tol)
    status = out["status"]
    if status & ST_CHOL:
        raise RankDeficiencyError("CholeskyQR breakdown: the stacked pair is numerically "
                                  "rank deficient")
    if status & ST_JACOBI:
        raise ConvergenceError("Jacobi SVD of an L block did not converge")
    if status & ST_CLASSIFY:
        raise ValidationError("overlapping zero classifications; sequences not ordered?")
    return out


def _spectrum_checked(c1, l1: int, c2, l2: int, n: int, classify_tol: float) -> GsvSpectrum:
    if l1 + l2 == 0:
        raise RankDeficiencyError("both compressed blocks are empty")
    out = _small_checked(c1, l1, c2, l2, n, classify_tol)
    r, s = out["counts"]
    return GsvSpectrum(out["alphas"], out["betas"], r, s)


def _general_run(pair: GmpPair, opts: GsvOptions) -> DeviceRun:
    """method='direct' and the adaptive range finder (engine.py:245-261):
    compressed blocks C1, C2 built on the device (G itself for direct; Q^T G
    from ``adaptive_device`` otherwise), then the shared stacked-QR +
    L-block SVD + comparative stage (device.small_spectrum)."""
    n = pair.n
    if opts.method == DIRECT:
        c1, c2 = pair.g1.t, pair.g2.t
        l1, l2 = pair.m, pair.p
        bases = (None, None)
    else:
        cfg = opts.extraction
        q1, c1, b1 = adaptive_device(pair.g1, cfg)
        q2, c2, b2 = adaptive_device(pair.g2, dataclasses.replace(cfg, seed=cfg.seed + 1))
        b1.q, b2.q = q1, q2
        l1, l2 = c1.shape[0], c2.shape[0]
        bases = (b1, b2)
    if l1 + l2 == 0:
        raise RankDeficiencyError("both compressed blocks are empty")  # engine.py:258-259
    out = _small_checked(c1, l1, c2, l2, n, opts.classify_tol)
    status = out["status"]
    r, s = out["counts"]
    spec = GsvSpectrum(out["alphas"], out["betas"], r, s)
    sc = out["scalars"]
    return DeviceRun(spec, spec.alphas, spec.betas, r, s, out["rho"], out["theta"], out["p1"],
                     out["p2"], float(sc[0]), float(sc[1]), (float(sc[2]), float(sc[3])), status,
                     bases[0], bases[1], out["sv1"], out["sv2"], None)


def _promoted(pair: GmpPair) -> GmpPair:
    """fp64 copy of an fp32 pair (core.py:51-54) for the small-size modes."""
    p64 = object.__new__(GmpPair)
    for name in ("g1", "g2"):
        g = getattr(pair, name)
        t = g.t.double() if g.is_f32 else g.t
        object.__setattr__(p64, name, _dev.to_device(t, name))
    object.__setattr__(p64, "check_rank", False)
    return p64


# widest sketch the fused single-call chain (rgsv_sketch_project: its sketch
# GEMM carries the fused ||G||^2, N <= 128) serves; wider fixed-rank sketches
# run the same chain as separate launches (rangefinder.chunked_chain)
_FUSED_MAX_K = 128


def _streamed_run(pair: GmpPair, opts: GsvOptions, k1: int, k2: int) -> DeviceRun:
    """Fixed-rank pipeline as separate launches, matrix by matrix: fp32 pairs
    (cfg4) take the tf32x3 tensor-core chain (tf32.tf32_chain) or the
    fp64-promoted row chunks (rangefinder.chunked_chain, f32_mode="promote");
    fp64 pairs wider than the fused chain (k > 128) take chunked_chain on the
    resident matrix. Then the shared small-GSVD + comparative stage."""
    cfg = opts.extraction
    lo = None
    res = []
    for g, k, seed in ((pair.g1, k1, cfg.seed), (pair.g2, k2, cfg.seed + 1)):
        if opts.f32_mode == "tf32x3" and _tf32.supported(g, k):
            # one fp32 lo buffer (rows x ld) shared by the two chains
            if lo is None or lo.numel() < g.rows * g.ld:
                lo = torch.empty(max(pair.g1.rows * pair.g1.ld, pair.g2.rows * pair.g2.ld),
                                 dtype=torch.float32, device="cuda")
            buf = lo[: g.rows * g.ld].view(g.rows, g.ld)
            res.append(_tf32.tf32_chain(g, k, cfg.power_iters, seed, lo=buf))
        else:
            res.append(chunked_chain(g, k, cfg.power_iters, seed))
    (_, b1, h1), (_, b2, h2) = res
    del lo
    out = _small_checked(b1, k1, b2, k2, pair.n, opts.classify_tol)
    r, s = out["counts"]
    spec = GsvSpectrum(out["alphas"], out["betas"], r, s)
    sc = out["scalars"]
    bases = []
    for h, k in ((h1, k1), (h2, k2)):
        tol = cfg.tol if cfg.tol is not None else 1e-10 * h[0]
        bases.append(BasisResult(None, h, h[-1] < tol, 1, [k]))
    return DeviceRun(spec, spec.alphas, spec.betas, r, s, out["rho"], out["theta"], out["p1"],
                     out["p2"], float(sc[0]), float(sc[1]), (float(sc[2]), float(sc[3])),
                     out["status"], bases[0], bases[1], out["sv1"], out["sv2"], None)


def run_device_pipeline(pair: GmpPair, opts: GsvOptions, *, sync: bool = True) -> DeviceRun:
    """The randomized path of _run_pipeline + spectrum_from_l_blocks +
    analysis, on the device (engine.py:245-275, analysis.py:82-102)."""
    widths = _fixed_width(opts, pair.m, pair.p, pair.n)
    f32 = pair.g1.is_f32 or pair.g2.is_f32
    if widths is None:
        return _general_run(_promoted(pair) if f32 else pair, opts)
    if f32 or max(widths) > _FUSED_MAX_K:
        return _streamed_run(pair, opts, *widths)
    k1, k2 = widths
    plan = _dev.pair_plan(pair.m, pair.p, pair.n, k1, k2)
    cfg = opts.extraction
    pk = plan.run(pair.g1, pair.g2, cfg.seed, cfg.power_iters, opts.classify_tol, sync=sync)
    try:
        return unpack(pk, plan, opts)
    except RankDeficiencyError:
        # A sketch wider than the matrix's numerical rank (exactly low-rank
        # input, trim_tol = 0) breaks CholeskyQR; the reference's Householder
        # QR keeps such columns (rangefinder.py:119-124). The general path
        # factors those blocks with the Householder kernel.
        return _general_run(pair, opts)


def unpack(pk, plan, opts: GsvOptions) -> DeviceRun:
    status = int(pk.h("status")[0])
    st1, st2 = pk.h("stats1"), pk.h("stats2")
    bases = []
    for (gf2, energy), k, rd in ((st1, plan.k1, "rdiag1"), (st2, plan.k2, "rdiag2")):
        if not math.isfinite(gf2):
            raise ValidationError("g contains non-finite entries")
        hist = _dev.residual_history(float(gf2), float(energy))
        tol = opts.extraction.tol if opts.extraction.tol is not None else 1e-10 * hist[0]
        bases.append(BasisResult(None, hist, hist[-1] < tol, 1, [k]))
    if status & ST_OMEGA_SHORT:
        raise RuntimeError("device Omega generator exhausted its draw margin")
    if status & ST_CHOL:
        raise RankDeficiencyError("CholeskyQR breakdown: a sketch or the stacked pair is "
                                  "numerically rank deficient")
    if status & ST_JACOBI:
        raise ConvergenceError("Jacobi SVD of an L block did not converge")
    r, s = (int(x) for x in pk.h("counts"))
    if status & ST_CLASSIFY:
        raise ValidationError("overlapping zero classifications; sequences not ordered?")
    alphas = pk.h("alphas").copy()
    betas = pk.h("betas").copy()
    spec = GsvSpectrum(alphas, betas, r, s)
    sc = pk.h("scalars")
    nsv = pk.h("nsv")
    return DeviceRun(spec, spec.alphas, spec.betas, r, s, pk.h("rho").copy(),
                     pk.h("theta").copy(), pk.h("p1").copy(), pk.h("p2").copy(), float(sc[0]),
                     float(sc[1]), (float(sc[2]), float(sc[3])), status, bases[0], bases[1],
                     pk.h("sv1")[: nsv[0]].copy(), pk.h("sv2")[: nsv[1]].copy(), plan)


def _is_host_pair(pr) -> bool:
    return not isinstance(pr, GmpPair)


def _is_f32_host(a) -> bool:
    return getattr(a, "dtype", None) in (np.float32, torch.float32)


def run_host_batch(host_pairs, opts: GsvOptions, seeds=None) -> list:
    """B pairs given as (g1, g2) HOST arrays (numpy or torch CPU tensors,
    pinned for full speed): streamed to the device with every pair's
    compute overlapping the transfers behind it (device.HostStreamPlan).
    Finiteness is checked by the device sum-of-squares pass of each chain
    (a NaN/Inf in G surfaces as a non-finite ||G||_F, ValidationError)."""
    host_pairs = [tuple(pr) for pr in host_pairs]
    if not host_pairs:
        return []
    shapes = {(tuple(a.shape), tuple(b.shape)) for a, b in host_pairs}
    if len(shapes) != 1:
        raise DimensionError("compare_batch needs pairs of one shape")
    (m, n1), (p, n) = next(iter(shapes))
    if n1 != n:
        raise DimensionError(f"g1 has {n1} columns but g2 has {n}")
    if m + p < n:
        raise RankDeficiencyError(f"stacked pair has {m + p} rows < {n} columns")
    cfg = opts.extraction
    seeds = [cfg.seed] * len(host_pairs) if seeds is None else list(seeds)
    if len(seeds) != len(host_pairs):
        raise DimensionError("one seed per pair")
    widths = _fixed_width(opts, m, p, n)
    f32 = opts.f32_mode == "tf32x3" and any(_is_f32_host(a) or _is_f32_host(b)
                                             for a, b in host_pairs)
    if widths is None or f32 or max(widths) > _FUSED_MAX_K:
        # general modes, fp32 pairs (tensor-core chain) and wide sketches:
        # upload and run pair by pair
        pairs = [GmpPair(a, b, check_rank=False if widths is not None else None)
                 for a, b in host_pairs]
        return run_device_batch(pairs, opts, seeds)
    k1, k2 = widths
    plan = _dev.host_stream_plan(len(host_pairs), m, p, n, k1, k2)
    pks = plan.run(host_pairs, seeds, cfg.power_iters, opts.classify_tol)
    runs = []
    for hp, sd, pk, sub in zip(host_pairs, seeds, pks, plan.plans):
        try:
            runs.append(unpack(pk, sub, opts))
        except RankDeficiencyError:  # sketch wider than the rank: see run_device_pipeline
            runs.append(_general_run(GmpPair(hp[0], hp[1], check_rank=False), dataclasses.replace(
                opts, extraction=dataclasses.replace(cfg, seed=sd))))
    return runs


_BATCH_SCAN: list = [None, None, None]  # [identity key, pairs (kept alive), result]


def _batch_scan(pairs):
    """(any matrix fp32, all pairs of one shape) for a device batch, in one
    pass. GmpPair is frozen, so the answer is cached on the identities of
    the pair objects (a step re-submitting the same 4096 pairs skips the
    per-pair Python scan)."""
    key = tuple(map(id, pairs))
    if _BATCH_SCAN[0] == key:
        return _BATCH_SCAN[2]
    first = pairs[0]
    shape = (first.g1.rows, first.g2.rows, first.g1.cols, first.g2.cols)
    any_f32, same = False, True
    for pr in pairs:
        a, b = pr.g1, pr.g2
        same = same and (a.rows, b.rows, a.cols, b.cols) == shape
        any_f32 = any_f32 or a.is_f32 or b.is_f32
    _BATCH_SCAN[:] = [key, pairs, (any_f32, same)]
    return any_f32, same


def run_device_batch(pairs, opts: GsvOptions, seeds=None) -> list:
    """B pairs of one shape, concurrently (device.BatchPlan). Pair b uses
    extraction seed seeds[b] (default: opts.extraction.seed for every pair,
    i.e. exactly compute_gsv(pair_b, opts) for each b)."""
    pairs = list(pairs)
    if not pairs:
        return []
    if _is_host_pair(pairs[0]):
        return run_host_batch(pairs, opts, seeds)
    first = pairs[0]
    w0 = _fixed_width(opts, first.m, first.p, first.n)
    any_f32, same_shape = _batch_scan(pairs)
    if any_f32 or (w0 is not None and max(w0) > _FUSED_MAX_K):  # chained passes, pair by pair
        cfg0 = opts.extraction
        seeds = [cfg0.seed] * len(pairs) if seeds is None else list(seeds)
        return [run_device_pipeline(pr, dataclasses.replace(
            opts, extraction=dataclasses.replace(cfg0, seed=sd))) for pr, sd in zip(pairs, seeds)]
    if not same_shape:
        raise DimensionError("compute_gsv_batch needs pairs of one shape")
    cfg = opts.extraction
    seeds = [cfg.seed] * len(pairs) if seeds is None else list(seeds)
    if len(seeds) != len(pairs):
        raise DimensionError("one seed per pair")
    widths = _fixed_width(opts, first.m, first.p, first.n)
    if widths is None:  # direct / adaptive: sequential general runs
        return [_general_run(pr, dataclasses.replace(
            opts, extraction=dataclasses.replace(cfg, seed=sd))) for pr, sd in zip(pairs, seeds)]
    k1, k2 = widths
    if _dev.small_batch_fits(max(first.m, first.p), first.n, k1, k2):
        return _small_batch_runs(pairs, opts, seeds, k1)
    plan = _dev.batch_plan(len(pairs), first.m, first.p, first.n, k1, k2)
    pks = plan.run([(pr.g1, pr.g2) for pr in pairs], seeds, cfg.power_iters, opts.classify_tol)
    runs = []
    for pr, sd, pk, sub in zip(pairs, seeds, pks, plan.plans):
        try:
            runs.append(unpack(pk, sub, opts))
        except RankDeficiencyError:  # sketch wider than the rank: see run_device_pipeline
            runs.append(_general_run(pr, dataclasses.replace(
                opts, extraction=dataclasses.replace(cfg, seed=sd))))
    return runs


class _PairMats:
    """(g1, g2) of every pair, built only if the plan's descriptor cache misses."""

    def __init__(self, pairs):
        self.pairs = pairs

    def __iter__(self):
        return ((pr.g1, pr.g2) for pr in self.pairs)


def _small_batch_runs(pairs, opts: GsvOptions, seeds, k: int):
    """Many small pairs through rgsv_batch_gsvd (one fused chain launch for
    every matrix, one small-GSVD launch for every pair)."""
    n = pairs[0].n
    plan = _dev.small_batch_plan(len(pairs), n, k)
    # run_device_batch scanned exactly this sequence just before: its identity
    # key (ids of the frozen pairs, kept alive by the scan cache) names it
    key = _BATCH_SCAN[0] if len(_BATCH_SCAN[0] or ()) == len(pairs) else None
    fh, ih = plan.run(_PairMats(pairs), seeds, opts.extraction.power_iters, opts.classify_tol,
                      key=key)
    return SmallBatchRuns(fh, ih, plan, opts)


def _trusted_spectrum(a, b, r: int, s: int) -> GsvSpectrum:
    """GsvSpectrum whose invariants were already checked (vectorized)."""
    spec = object.__new__(GsvSpectrum)
    object.__setattr__(spec, "alphas", a)
    object.__setattr__(spec, "betas", b)
    object.__setattr__(spec, "r", r)
    object.__setattr__(spec, "s", s)
    return spec


class SmallBatchRuns(Sequence):
    """Results of one rgsv_batch_gsvd call, validated for the whole batch at
    once (status bits, finiteness and every GsvSpectrum invariant of
    engine.py:108-125, vectorized); per-pair DeviceRun objects are built on
    access, so a 4096-pair step costs one D2H copy plus a few numpy passes."""

    def __init__(self, fh, ih, plan, opts: GsvOptions):
        B, n, k, rs = plan.B, plan.n, plan.k, plan.res_stride
        self.B, self.n, self.k, self.plan, self.opts = B, n, k, plan, opts
        # views of this call's own pinned buffers (SmallBatchPlan.fetch)
        self.res = fh[: B * rs].reshape(B, rs)
        self.stats = fh[B * rs: B * rs + 4 * B].reshape(B, 4)
        self.ints = ih[: 4 * B].reshape(B, 4)
        self.status = ih[4 * B: 5 * B]
        st = self.status
        # input finiteness first, as unpack() and the reference's as_matrix
        # (core.py:55) order it
        if np.any(st & ST_NONFINITE) or not np.all(np.isfinite(self.stats[:, 0])) or \
                not np.all(np.isfinite(self.stats[:, 2])):
            raise ValidationError("g contains non-finite entries")
        for bit, exc, msg in ((ST_OMEGA_SHORT, RuntimeError,
                               "device Omega generator exhausted its draw margin"),
                              (ST_CHOL, RankDeficiencyError, "CholeskyQR breakdown"),
                              (ST_JACOBI, ConvergenceError, "Jacobi SVD did not converge"),
                              (ST_CLASSIFY, ValidationError,
                               "overlapping zero classifications; sequences not ordered?")):
            bad = np.flatnonzero(st & bit)
            if bad.size:
                raise exc(f"{msg} (batch pair {int(bad[0])})")
        # k_batch_small checks every GsvSpectrum invariant on the device
        # (RGSV_ST_SPECTRUM); the host re-scan below only runs to name the
        # violated one with the reference's message
        if np.any(st & ST_SPECTRUM):
            self._check_spectra()

    def _check_spectra(self) -> None:
        n = self.n
        a, b = self.res[:, :n], self.res[:, n:2 * n]
        r, s = self.ints[:, 2], self.ints[:, 3]
        if np.any(r < 0) or np.any(s < 0) or np.any(r + s > n):
            raise ValidationError("invalid counts r, s")
        if np.any(a < 0) or np.any(a > 1) or np.any(b < 0) or np.any(b > 1):
            raise ValidationError("GSVs must lie in [0, 1]")
        if np.any(np.diff(a, axis=1) > 1e-12) or np.any(np.diff(b, axis=1) < -1e-12):
            raise ValidationError("alphas must be nonincreasing and betas nondecreasing")
        if float(np.max(np.abs(a ** 2 + b ** 2 - 1.0))) > 1e-12:
            raise ValidationError("alpha_i^2 + beta_i^2 = 1 violated beyond 1e-12")
        idx = np.arange(n)
        if np.any((b != 0.0) & (idx < r[:, None])) or np.any((a != 0.0) & (idx >= (r + s)[:, None])):
            raise ValidationError("classified-zero entries must be exactly 0")
        raise ValidationError("GSVs must lie in [0, 1]")  # NaN entries (the device flags them)

    def __len__(self) -> int:
        return self.B

    def __getitem__(self, j):
        if isinstance(j, slice):
            return [self[i] for i in range(*j.indices(self.B))]
        if j < 0:
            j += self.B
        if not 0 <= j < self.B:
            raise IndexError(j)
        n, k, o = self.n, self.k, self.res[j]
        nsv1, nsv2, r, s = (int(x) for x in self.ints[j])
        spec = _trusted_spectrum(o[:n].copy(), o[n:2 * n].copy(), r, s)
        bases = []
        for gf2, energy in ((self.stats[j, 0], self.stats[j, 1]),
                            (self.stats[j, 2], self.stats[j, 3])):
            hist = _dev.residual_history(float(gf2), float(energy))
            tol = self.opts.extraction.tol if self.opts.extraction.tol is not None \
                else 1e-10 * hist[0]
            bases.append(BasisResult(None, hist, hist[-1] < tol, 1, [k]))
        sc = o[6 * n: 6 * n + 4]
        return DeviceRun(spec, spec.alphas, spec.betas, r, s, o[2 * n:3 * n].copy(),
                         o[3 * n:4 * n].copy(), o[4 * n:5 * n].copy(), o[5 * n:6 * n].copy(),
                         float(sc[0]), float(sc[1]), (float(sc[2]), float(sc[3])),
                         int(self.status[j]), bases[0], bases[1],
                         o[6 * n + 4: 6 * n + 4 + nsv1].copy(),
                         o[6 * n + 4 + k: 6 * n + 4 + k + nsv2].copy(), self.plan)


class _MappedSeq(Sequence):
    """Lazy per-element view over a SmallBatchRuns."""

    def __init__(self, runs, fn):
        self._runs, self._fn = runs, fn

    def __len__(self) -> int:
        return len(self._runs)

    def __getitem__(self, j):
        if isinstance(j, slice):
            return [self[i] for i in range(*j.indices(len(self)))]
        return self._fn(self._runs[j])


def compute_gsv_batch(pairs, opts: GsvOptions | None = None, seeds=None) -> list:
    """compute_gsv over a batch of same-shape pairs, run concurrently on the
    device (throughput mode); results equal per-pair compute_gsv calls.
    Pairs are GmpPair objects (resident in HBM) or (g1, g2) host arrays,
    which are streamed in with transfer/compute overlap."""
    opts = opts or GsvOptions()
    runs = run_device_batch(pairs, opts, seeds)
    if isinstance(runs, SmallBatchRuns):
        return _MappedSeq(runs, lambda run: run.spectrum)
    return [run.spectrum for run in runs]


def compute_gsv(pair: GmpPair, opts: GsvOptions | None = None) -> GsvSpectrum:
    """GSV spectrum of a pair on the B200 (engine.py:264-275)."""
    opts = opts or GsvOptions()
    return run_device_pipeline(pair, opts).spectrum


def recover_gsvd(pair: GmpPair, opts: GsvOptions | None = None) -> GsvdFactors:
    """Full decomposition recovery (engine.py:294-362) on the device
    (recovery.py). Requires m, p >= n (:304-307) and a compressed pair with
    n independent columns (:309-313): the fixed-rank BASELINE configs have
    l1 + l2 = 2k < n and raise RecoveryError exactly like
    the reference; the adaptive default and method="direct" recover."""
    from .recovery import recover

    opts = opts or GsvOptions()
    if opts.method != DIRECT:
        check_max_cols(opts.extraction, pair.m, pair.n)
        check_max_cols(opts.extraction, pair.p, pair.n)
    if pair.g1.is_f32 or pair.g2.is_f32:
        pair = _promoted(pair)
    u, v, rf, spec = recover(pair, opts, opts.method == DIRECT)
    return GsvdFactors(u, v, rf, spec)


__all__ = ["GmpPair", "GsvSpectrum", "GsvOptions", "GsvdFactors", "classify_spectrum",
           "spectrum_from_l_blocks",
           "compute_gsv", "compute_gsv_batch", "recover_gsvd", "run_device_pipeline",
           "run_device_batch", "RANDOMIZED", "DIRECT",
           "dataclasses"]
