"""Seeded parity sweep: random shapes, ranks, noise levels and modes (fixed
rank with q = 0..2, direct, the reference-default adaptive Alg. 1) through
the public API on the device, against the CPU oracle. The GSV tolerance is
conditioning-scaled (the pair's GSVs move by eps * cond(stacked pair) between
two backward-stable implementations: LAPACK in the oracle, the kernels here).

Adaptive cases whose stop test sits at the rounding floor are ill-posed in
the reference itself (residual = sqrt(max(|G|^2 - captured, 0)) against
tol = 1e-10 |G|: either exactly 0 or ~1e-8 |G| by one-ulp differences,
DESIGN.md section 2): those are recognised by the oracle's and the device's
block widths differing, counted, and excluded from the value comparison --
the sweep requires that they stay the minority."""
import numpy as np
import pytest

import paper_2404_09459_b200 as rg
from oracle import rgsv_oracle as orc

pytestmark = pytest.mark.gpu
EPS = 2.220446049250313e-16


def make_pair(rng, m, p, n, s, noise):
    """Two low-rank-plus-noise matrices sharing half of their right factor."""
    b1 = rng.standard_normal((n, s))
    sh = s // 2
    b2 = np.hstack([b1[:, :sh], rng.standard_normal((n, s - sh))])
    d = 10.0 ** (-2.0 * np.arange(s) / max(s, 1))
    g1 = (rng.standard_normal((m, s)) * d) @ b1.T + noise * rng.standard_normal((m, n))
    g2 = (rng.standard_normal((p, s)) * d) @ b2.T + noise * rng.standard_normal((p, n))
    return g1, g2


def draw_case(rng):
    n = int(rng.integers(3, 260))
    m = int(rng.integers(max(2, n // 3), 1200))
    p = int(rng.integers(max(2, n // 3), 1200))
    if m + p < n:
        m = n
    s = int(rng.integers(1, max(2, min(m, p, n) // 2 + 1)))
    noise = float(rng.choice([1e-3, 1e-6, 1e-9]))
    mode = str(rng.choice(["fixed", "fixed", "direct", "adaptive"]))
    seed = int(rng.integers(0, 1000))
    g1, g2 = make_pair(rng, m, p, n, s, noise)
    k = q = None
    if mode == "fixed":
        k = min(int(rng.integers(1, min(m, p, n) + 1)), 200)
        q = int(rng.integers(0, 3))
    return g1, g2, mode, seed, k, q


@pytest.mark.parametrize("sweep_seed", [1, 2])
def test_random_pairs_vs_oracle(sweep_seed):
    rng = np.random.default_rng(sweep_seed)
    adaptive = floor_cases = 0
    for idx in range(40):
        g1, g2, mode, seed, k, q = draw_case(rng)
        tag = f"sweep {sweep_seed} case {idx}: {g1.shape} {g2.shape} {mode} seed={seed} k={k} q={q}"
        pair = rg.GmpPair(g1, g2)
        sv = np.linalg.svd(np.vstack([g1, g2]), compute_uv=False)
        tol = max(1e-11, 200.0 * EPS * sv[0] / sv[-1])
        if mode == "fixed":
            opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(k, seed, q))
            o = orc.run_pipeline(g1, g2, k=k, q=q, seed=seed)
        elif mode == "direct":
            opts = rg.GsvOptions(method="direct")
            o = orc.run_pipeline(g1, g2, direct=True)
        else:
            adaptive += 1
            opts = rg.GsvOptions(extraction=rg.ExtractionConfig(seed=seed))
            o = orc.run_pipeline(g1, g2, seed=seed)
            pl = rg.engine._run_pipeline(pair, opts)
            widths = (pl.l1_block.shape[0], pl.l2_block.shape[0])
            if widths != (o.l1_block.shape[0], o.l2_block.shape[0]):
                floor_cases += 1  # the reference's own coin flip (docstring)
                continue
        spec = rg.compute_gsv(pair, opts)
        assert (spec.r, spec.s) == (o.r, o.s), tag
        assert np.max(np.abs(spec.alphas - o.alphas)) <= tol, tag
        assert np.max(np.abs(spec.betas - o.betas)) <= tol, tag
    assert floor_cases <= adaptive // 2, (floor_cases, adaptive)
