"""Comparative-analysis quantities (reference ``rgsv/analysis.py``).

``compare`` runs the whole pipeline on the B200 and reads rho, theta,
P1/P2 and D1/D2 from the fused comparative kernel of the same run
(k_comparative, csrc/small.cu), so no per-index arithmetic happens on the
host. The per-quantity helpers accept a ``GsvSpectrum`` like the
reference's and evaluate through the same device kernel.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import device as _dev
from ._native import ST_DEGENERATE, ST_NOT_NORMALIZED, check, lib
from .engine import (
    GmpPair,
    GsvOptions,
    GsvSpectrum,
    SmallBatchRuns,
    _MappedSeq,
    run_device_batch,
    run_device_pipeline,
)
from .errors import DegenerateSpectrumError, ValidationError

QUARTER_PI = math.pi / 4


@dataclass(frozen=True)
class ComparativeReport:
    """analysis.py:22-34."""

    spectrum: GsvSpectrum
    rho: np.ndarray
    theta: np.ndarray
    p1: np.ndarray
    p2: np.ndarray
    d1: float
    d2: float
    meta: dict = field(default_factory=dict)


def _spectrum_quantities(spec: GsvSpectrum):
    """rho, theta, p1, p2, (d1, d2), (sum p1, sum p2), status of a given
    spectrum through the device kernel (rgsv_spectrum_quantities)."""
    n = spec.n
    a = torch.from_numpy(np.ascontiguousarray(spec.alphas)).cuda()
    b = torch.from_numpy(np.ascontiguousarray(spec.betas)).cuda()
    out = torch.zeros(4 * n + 4, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = _dev.sp(torch.cuda.current_stream())
    rc = lib().rgsv_spectrum_quantities(
        _dev.vp(a), _dev.vp(b), n, int(spec.r), _dev.vp(out[0:n]), _dev.vp(out[n:2 * n]),
        _dev.vp(out[2 * n:3 * n]), _dev.vp(out[3 * n:4 * n]), _dev.vp(out[4 * n:]),
        _dev.vp(status), st)
    check(rc, "rgsv_spectrum_quantities")
    h = out.cpu().numpy()
    return (h[0:n].copy(), h[n:2 * n].copy(), h[2 * n:3 * n].copy(), h[3 * n:4 * n].copy(),
            (float(h[4 * n]), float(h[4 * n + 1])), (float(h[4 * n + 2]), float(h[4 * n + 3])),
            int(status.item()))


def relative_significance(spec: GsvSpectrum) -> np.ndarray:
    """alpha/beta, +inf where beta is classified zero (analysis.py:37-42)."""
    return _spectrum_quantities(spec)[0]


def angular_distances(spec: GsvSpectrum) -> np.ndarray:
    """atan2(alpha, beta) - pi/4 (analysis.py:45-51)."""
    return _spectrum_quantities(spec)[1]


def eigenexpression_fractions(spec: GsvSpectrum) -> tuple[np.ndarray, np.ndarray]:
    """Normalized squared GSVs (analysis.py:54-60)."""
    q = _spectrum_quantities(spec)
    if q[6] & ST_DEGENERATE:
        raise DegenerateSpectrumError("spectrum has vanishing alpha- or beta-energy")
    return q[2], q[3]


def shannon_entropy(p) -> float:
    """Normalized Shannon entropy (analysis.py:63-79), reduced on the device."""
    v = np.asarray(p, dtype=np.float64)
    if v.ndim != 1 or v.size < 2:
        raise ValidationError(
            f"need a 1-D probability vector of length >= 2, got shape {v.shape}")
    if np.any(v < 0):
        raise ValidationError("probability vector has negative entries")
    dev = torch.from_numpy(np.ascontiguousarray(v)).cuda()
    out = torch.zeros(4, dtype=torch.float64, device="cuda")
    rc = lib().rgsv_entropy(_dev.vp(dev), v.size, _dev.vp(out),
                            _dev.sp(torch.cuda.current_stream()))
    check(rc, "rgsv_entropy")
    d, _, total, _ = (float(x) for x in out.cpu().tolist())
    if abs(total - 1.0) > 1e-10:
        raise ValidationError(f"probability vector sums to {total!r}, not 1")
    return d


def _report(run, opts: GsvOptions) -> ComparativeReport:
    if run.status & ST_DEGENERATE:
        raise DegenerateSpectrumError("spectrum has vanishing alpha- or beta-energy")
    if run.status & ST_NOT_NORMALIZED:
        raise ValidationError("eigenexpression fractions do not sum to 1")
    meta = {
        "method": opts.method,
        "seed": opts.extraction.seed,
        "tol": opts.extraction.tol,
        "classify_tol": opts.classify_tol,
    }
    return ComparativeReport(spectrum=run.spectrum, rho=run.rho, theta=run.theta, p1=run.p1,
                             p2=run.p2, d1=run.d1, d2=run.d2, meta=meta)


def compare_batch(pairs, opts: GsvOptions | None = None, seeds=None) -> list:
    """compare over a batch of same-shape pairs run concurrently on the
    device (throughput mode); equal to per-pair compare calls."""
    opts = opts or GsvOptions()
    runs = run_device_batch(pairs, opts, seeds)
    if isinstance(runs, SmallBatchRuns):
        st = runs.status
        if np.any(st & ST_DEGENERATE):
            raise DegenerateSpectrumError("spectrum has vanishing alpha- or beta-energy")
        if np.any(st & ST_NOT_NORMALIZED):
            raise ValidationError("eigenexpression fractions do not sum to 1")
        return _MappedSeq(runs, lambda run: _report(run, opts))
    return [_report(run, opts) for run in runs]


def compare(pair: GmpPair, opts: GsvOptions | None = None) -> ComparativeReport:
    """Spectrum + every comparison quantity, one device run
    (analysis.py:82-102)."""
    opts = opts or GsvOptions()
    return _report(run_device_pipeline(pair, opts), opts)


__all__ = ["ComparativeReport", "relative_significance", "angular_distances",
           "eigenexpression_fractions", "shannon_entropy", "compare", "compare_batch",
           "QUARTER_PI"]
