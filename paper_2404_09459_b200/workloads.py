"""Synthetic matrix pairs with the BASELINE.json config shapes.

The reference ships no generator for these configs; this
is the builder-owned, deterministic generator specified there:

    rng = default_rng(data_seed); draw in order A1 (m x s), A2 (p x s),
    B1 (n x s), B2 = [B1[:, :shared], new n x (s - shared)], E1 (m x n),
    E2 (p x n), all N(0, 1);  d_j = 10^(-c j / s);
    G_i = (A_i diag d) B_i^T + eps E_i.

Ω is not drawn here: it follows the reference convention (extraction
seed for G1, seed + 1 for G2; ``rangefinder.py:101,112``,
``engine.py:252-253``). The paper's genome datasets are not available
(no network); these seeded pairs stand in for them with the configs'
shapes, ranks, shared-signal structure and noise levels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class PairConfig:
    name: str
    m: int
    p: int
    n: int
    s: int
    shared: int
    decay: float  # c in d_j = 10^(-c j / s)
    eps: float
    k: int
    q: int
    dtype: str = "f64"
    batch: int = 1
    data_seed: int = 1_000_003

    @property
    def flops(self) -> float:
        """Algorithmic GEMM flops per pair: 2 (m + p) n k (2q + 2)
        (SURVEY.md §8 table)."""
        return 2.0 * (self.m + self.p) * self.n * self.k * (2 * self.q + 2)

    @property
    def g_bytes(self) -> int:
        w = 8 if self.dtype == "f64" else 4
        return w * (self.m + self.p) * self.n

    @property
    def stream_bytes(self) -> float:
        """Algorithmic bytes per pair: one read of G per GEMM pass."""
        return float(self.g_bytes) * (2 * self.q + 2)


# BASELINE.json "configs", in order.
CONFIGS = {
    "cfg0": PairConfig("cfg0", 2000, 1500, 200, 20, 10, 0.0, 1e-8, 30, 1),
    "cfg1": PairConfig("cfg1", 20000, 16000, 1000, 50, 25, 2.0, 1e-8, 60, 2),
    "cfg2": PairConfig("cfg2", 200000, 150000, 4000, 100, 50, 3.0, 1e-8, 120, 2),
    "cfg3": PairConfig("cfg3", 4000, 3000, 64, 8, 4, 0.0, 1e-8, 16, 1, batch=4096),
    "cfg4": PairConfig("cfg4", 1_000_000, 800_000, 8192, 256, 128, 2.0, 1e-4, 288, 1,
                       dtype="f32"),
}


def make_pair(cfg: PairConfig, data_seed: int | None = None, m: int | None = None,
              p: int | None = None, n: int | None = None):
    """Host-side (numpy, float64) pair for ``cfg``; shape overrides allow
    reduced-size instances with the same structure."""
    seed = cfg.data_seed if data_seed is None else data_seed
    m = cfg.m if m is None else m
    p = cfg.p if p is None else p
    n = cfg.n if n is None else n
    rng = np.random.default_rng(seed)
    a1 = rng.standard_normal((m, cfg.s))
    a2 = rng.standard_normal((p, cfg.s))
    b1 = rng.standard_normal((n, cfg.s))
    b2 = np.hstack([b1[:, : cfg.shared], rng.standard_normal((n, cfg.s - cfg.shared))])
    e1 = rng.standard_normal((m, n))
    e2 = rng.standard_normal((p, n))
    d = 10.0 ** (-cfg.decay * np.arange(cfg.s) / cfg.s)
    g1 = (a1 * d) @ b1.T + cfg.eps * e1
    g2 = (a2 * d) @ b2.T + cfg.eps * e2
    return g1, g2


def batch_seeds(j: int):
    """cfg3 per-pair seeds: data seed j, extraction (Ω) seed 2j, so pair j's
    G2 stream (2j + 1) never collides with pair j+1's G1 stream."""
    return j, 2 * j
