"""Synthetic pairs with a known GSV spectrum (reference ``rgsv/synthetic.py``).

The generator feeds the timing harness (``bench.py`` of this package) and the
accuracy tests either side of the hot path. The random draws come from
numpy's seeded PCG64 stream in the reference's order (interior GSVs, shared
right factor, then the two left blocks: synthetic.py:84-99), so a seed names
the same pair here and there; the linear algebra runs on the B200 through
this package's own kernels -- ``core.reduced_qr`` for the orthonormal left
blocks (synthetic.py:102-103), the DMMA ``rgsv_gemm_gx`` for the two products
(synthetic.py:106-107) and the device Jacobi (values only) for cond(R*)
(synthetic.py:109).
The pair matches the reference's to rounding (the QR kernels are not LAPACK's);
the true spectrum is bit-identical.

Only the real field runs on the B200 path: ``field="complex"`` (the
reference's default) is accepted by ``SynthSpec`` for interface parity and
rejected by ``synth_gmp`` with ValidationError, like every complex input of
this package (no CPU fallback).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import core
from . import device as _dev
from .engine import GmpPair, GsvSpectrum
from .errors import InfeasibleRankError, ValidationError

_SEED_MASK = (1 << 64) - 1


@dataclass(frozen=True)
class SynthSpec:
    """Shape, rank fraction, seed and field of a synthetic pair
    (synthetic.py:22-49). Each matrix has rank floor(rank_frac * min(m, p, n));
    the interior GSVs are sorted uniform draws on (0, 1)."""

    m: int
    p: int
    n: int
    rank_frac: float = 0.6
    seed: int = 0
    field: str = core.COMPLEX

    def __post_init__(self):
        if self.m < 1 or self.p < 1:
            raise ValidationError(f"m and p must be >= 1, got ({self.m}, {self.p})")
        if self.n < 2:
            raise ValidationError(f"n must be >= 2, got {self.n}")
        if not 0 < self.rank_frac <= 1:
            raise ValidationError(f"rank_frac must be in (0, 1], got {self.rank_frac}")
        if self.field not in (core.REAL, core.COMPLEX):
            raise ValidationError(f"field must be 'real' or 'complex', got {self.field!r}")

    @property
    def rank(self) -> int:
        return int(math.floor(self.rank_frac * min(self.m, self.p, self.n)))


@dataclass(frozen=True)
class SynthResult:
    """The generated pair (resident in HBM), its exact spectrum and the
    condition number of the shared right factor (synthetic.py:52-60)."""

    pair: GmpPair
    true_spectrum: GsvSpectrum
    condition_r: float


def true_spectrum(n: int, rank: int, interior: np.ndarray) -> GsvSpectrum:
    """alpha = (1 .. 1, interior, 0 .. 0) with r = n - rank ones and
    n - rank zeros; beta completes it with exact 0 / 1 in the two outer
    blocks (synthetic.py:85-89)."""
    r = n - rank
    alphas = np.concatenate([np.ones(r), interior, np.zeros(n - rank)])
    betas = np.sqrt(1.0 - alphas**2)
    betas[:r] = 0.0
    betas[rank:] = 1.0
    return GsvSpectrum(alphas, betas, r=r, s=interior.size)


def _scaled_product(left: np.ndarray, scale: np.ndarray, right_rows: np.ndarray) -> torch.Tensor:
    """left (rows x k) @ (scale[:, None] * right_rows (k x n)) on the device:
    the row scaling is folded into the K-major right operand and the product
    runs on the DMMA GEMM (rgsv_gemm_gx)."""
    from .rangefinder import _Ops

    rows, k = left.shape
    n = right_rows.shape[1]
    a = _dev.to_device(left, "left factor")
    bt = _dev.to_device(np.ascontiguousarray((scale[:, None] * right_rows).T), "right factor")
    out = torch.zeros((rows, n + (n & 1)), dtype=torch.float64, device="cuda")
    _Ops().gx(_dev.vp(a.t), a.ld, _dev.vp(bt.t), bt.ld, _dev.vp(out), out.stride(0), rows, n, k)
    return out[:, :n]


def synth_gmp(spec: SynthSpec) -> SynthResult:
    """Generate a pair with known GSVs, deterministically per seed
    (synthetic.py:63-112). n - rank alphas and n - rank betas are exactly
    zero, which needs 2 * rank >= n (InfeasibleRankError otherwise)."""
    rank, n = spec.rank, spec.n
    if rank < 1:
        raise ValidationError(
            f"rank_frac {spec.rank_frac} with sizes ({spec.m}, {spec.p}, {spec.n}) "
            "yields empty matrices")
    n_interior = 2 * rank - n
    if n_interior < 0:
        raise InfeasibleRankError(
            f"rank {rank} per matrix cannot stack to full column rank {n}; "
            "increase rank_frac")
    if spec.field == core.COMPLEX:
        raise ValidationError("synth_gmp: complex pairs are not supported by the B200 path "
                              "(pass field='real')")
    _dev.require_device()

    rng = np.random.default_rng(int(spec.seed) & _SEED_MASK)
    interior = np.sort(rng.uniform(0.0, 1.0, n_interior))[::-1]
    spectrum = true_spectrum(n, rank, interior)
    r_star = rng.standard_normal((n, n))
    u_active = core.reduced_qr(rng.standard_normal((spec.m, rank))).q
    v_active = core.reduced_qr(rng.standard_normal((spec.p, rank))).q

    # nonzero alphas sit at indices [0, rank), nonzero betas at [n - rank, n)
    g1 = _scaled_product(u_active, spectrum.alphas[:rank], r_star[:rank])
    g2 = _scaled_product(v_active, spectrum.betas[n - rank:], r_star[n - rank:])

    # cond(R*) from the singular values alone (device Jacobi, no vectors)
    from .validation import _jacobi_values

    rd = _dev.to_device(r_star, "r_star")
    sr = _jacobi_values(rd.t.clone(), n, n)
    return SynthResult(GmpPair(g1, g2), spectrum, float(sr[0] / sr[-1]))


__all__ = ["SynthSpec", "SynthResult", "synth_gmp"]
