"""Timing harness: randomized vs direct GSV on the device path (reference
``rgsv/bench.py``). Same configuration object, record fields, seed rule and
summary as the reference, so scripts and the ``bench`` subcommand carry over;
what is timed is this package's ``engine._run_pipeline`` +
``engine.spectrum_from_l_blocks`` -- the seam bench.py:72-79 brackets -- with
the pair already resident in HBM (``GmpPair`` construction and file parsing
are outside the timed region, as in the reference). Both calls return host
arrays, so the device work has completed when the clock stops; a
``torch.cuda.synchronize()`` before the clock starts keeps earlier work out.

(The repository-level ``bench.py`` is the driver's throughput benchmark of
the BASELINE configurations; this module is the library's own harness.)
"""

from __future__ import annotations

import dataclasses
import statistics
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import engine
from .engine import DIRECT, RANDOMIZED, GmpPair, GsvOptions
from .errors import ValidationError
from .synthetic import SynthSpec, synth_gmp


@dataclass(frozen=True)
class RunConfig:
    """One run (bench.py:18-42): the pair comes from two matrix files or
    from the synthetic generator -- exactly one of the two -- plus the GSV
    options, the report destination / format and the repetition count."""

    g1_path: str | None = None
    g2_path: str | None = None
    synth: SynthSpec | None = None
    options: GsvOptions = field(default_factory=GsvOptions)
    output: str | None = None
    format: str = "csv"
    repetitions: int = 1

    def __post_init__(self):
        given = (self.g1_path is not None, self.g2_path is not None)
        if given[0] != given[1]:
            raise ValidationError("g1_path and g2_path must be given together")
        if all(given) == (self.synth is not None):
            raise ValidationError("exactly one input source: matrix files or synth spec")
        if self.repetitions < 1:
            raise ValidationError(f"repetitions must be >= 1, got {self.repetitions}")
        if self.format not in ("csv", "json"):
            raise ValidationError(f"format must be 'csv' or 'json', got {self.format!r}")


@dataclass(frozen=True)
class BenchRecord:
    """One timed repetition of one method (bench.py:45-61): wall seconds,
    spectrum error against the first direct run, final residuals and basis
    widths (None / full height for the direct method), pair shape."""

    method: str
    repetition: int
    seconds: float
    err_alpha: float
    err_beta: float
    residual1: float | None
    residual2: float | None
    l1: int
    l2: int
    m: int
    p: int
    n: int


def load_pair(cfg: RunConfig) -> GmpPair:
    """The pair a run configuration names, validated and placed in HBM
    (bench.py:64-70)."""
    if cfg.synth is not None:
        return synth_gmp(cfg.synth).pair
    from .io import read_matrix

    return GmpPair(read_matrix(cfg.g1_path), read_matrix(cfg.g2_path))


def _timed_run(pair: GmpPair, opts: GsvOptions):
    """(spectrum, pipeline, seconds) of one pass through the seam
    (bench.py:72-79)."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pl = engine._run_pipeline(pair, opts)
    spec = engine.spectrum_from_l_blocks(pl.l1_block, pl.l2_block, pair.n, opts.classify_tol)
    dt = time.perf_counter() - t0
    return spec, pl, dt


def _last_residual(basis):
    return None if basis is None else float(basis.residual_history[-1])


def run_bench(cfg: RunConfig) -> list[BenchRecord]:
    """Time both methods for ``cfg.repetitions`` repetitions each
    (bench.py:82-126). The direct method runs first; its first spectrum is
    the error reference of every record. Randomized repetition ``rep`` uses
    extraction seed ``base + rep``."""
    pair = load_pair(cfg)
    base = cfg.options
    records: list[BenchRecord] = []
    truth = None
    for method in (DIRECT, RANDOMIZED):
        for rep in range(cfg.repetitions):
            opts = dataclasses.replace(base, method=method)
            if method == RANDOMIZED:
                ext = dataclasses.replace(base.extraction, seed=base.extraction.seed + rep)
                opts = dataclasses.replace(opts, extraction=ext)
            spec, pl, dt = _timed_run(pair, opts)
            if truth is None:
                truth = spec
            records.append(BenchRecord(
                method=method, repetition=rep, seconds=dt,
                err_alpha=float(np.linalg.norm(spec.alphas - truth.alphas)),
                err_beta=float(np.linalg.norm(spec.betas - truth.betas)),
                residual1=_last_residual(pl.basis1), residual2=_last_residual(pl.basis2),
                l1=int(pl.l1_block.shape[0]), l2=int(pl.l2_block.shape[0]),
                m=pair.m, p=pair.p, n=pair.n))
    return records


def median_seconds(records: list[BenchRecord]) -> dict[str, float]:
    """Median wall time per method (bench.py:129-136)."""
    by_method: dict[str, list[float]] = {}
    for rec in records:
        by_method.setdefault(rec.method, []).append(rec.seconds)
    return {method: statistics.median(secs) for method, secs in by_method.items()}


__all__ = ["RunConfig", "BenchRecord", "load_pair", "run_bench", "median_seconds"]
