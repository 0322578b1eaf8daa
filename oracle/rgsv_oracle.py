"""numpy restatement of the reference rGSVD hot path (TEST INFRASTRUCTURE).

See ``oracle/__init__.py`` for who may import this and how it is pinned.
All citations are ``path:line`` under ``/root/reference/pkg/src/rgsv/``.
Power iterations (``power_iters`` > 0) are NOT in the reference
(SURVEY.md §0 F1); they are restated here as the standard subspace
iteration built from the reference's own primitives and are marked
"parity unpinned" wherever used.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED_MASK = (1 << 64) - 1
QUARTER_PI = math.pi / 4


# ----------------------------------------------------------------- core.py
def omega_block(rng: np.random.Generator, n: int, width: int, complex_field: bool = False):
    """One Gaussian sketch block drawn from a running stream
    (rangefinder.py:112-114; same convention as core.gaussian_matrix,
    core.py:60-76)."""
    om = rng.standard_normal((n, width))
    if complex_field:
        om = math.sqrt(0.5) * (om + 1j * rng.standard_normal((n, width)))
    return om


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """core.py:60-71 (real field)."""
    return np.random.default_rng(int(seed) & SEED_MASK).standard_normal((rows, cols))


def reduced_qr(a: np.ndarray):
    """Householder reduced QR with nonnegative real R diagonal
    (core.py:79-96)."""
    q, r = np.linalg.qr(a, mode="reduced")
    d = np.diagonal(r)
    if np.iscomplexobj(r):
        absd = np.abs(d)
        ph = np.where(absd > 0, d / np.where(absd > 0, absd, 1.0), 1.0)
    else:
        ph = np.where(d < 0.0, -1.0, 1.0)
    return q * ph, r * np.conj(ph)[:, None]


def sum_sq(a: np.ndarray) -> float:
    """Column sums of squared magnitudes combined with math.fsum
    (core.py:109-125)."""
    if a.size == 0:
        return 0.0
    sq = np.square(a.real) + np.square(a.imag) if np.iscomplexobj(a) else np.square(a)
    return float(math.fsum(np.atleast_1d(sq.sum(axis=0))))


def singular_values(block: np.ndarray) -> np.ndarray:
    """engine.py:228-231 / core.py:99-106: the reference takes the values
    from a full reduced SVD (gesdd with vectors), which is kept here so the
    values match it bit for bit."""
    if block.shape[0] == 0:
        return np.zeros(0)
    return np.linalg.svd(block, full_matrices=False)[1]


# ---------------------------------------------------------- rangefinder.py
@dataclass
class Basis:
    q: np.ndarray
    residual_history: list
    converged: bool
    iterations: int
    block_widths: list = field(default_factory=list)
    b: np.ndarray | None = None  # Q^H G of the final basis (engine.py:255)


def extract_basis(g, tol=None, blocksize=100, seed=0, max_cols=None, trim_tol=1e-12,
                  power_iters=0) -> Basis:
    """Alg. 1, rangefinder.py:68-135, plus (power_iters > 0, unpinned)
    per-block subspace iteration Y <- G qr(G^H qr(Y).q).q re-projected
    against the current basis like the raw sketch (rangefinder.py:116-118).
    At power_iters == 0 this is the reference statement by statement."""
    a = np.asarray(g)
    m, n = a.shape
    gf2 = sum_sq(a)                                        # rangefinder.py:83
    normf = math.sqrt(gf2)
    tol = tol if tol is not None else 1e-10 * normf        # :85
    trim_cut = trim_tol * normf                            # :86
    q = np.zeros((m, 0), dtype=a.dtype)                    # :93
    history = [normf]
    widths = []
    if normf == 0.0 or normf < tol:                        # :96
        return Basis(q, history, True, 0, widths)
    b = min(blocksize, n)                                  # :99
    nblocks = -(-n // b)
    rng = np.random.default_rng(int(seed) & SEED_MASK)     # :101
    captured = []
    converged = False
    iterations = 0
    cplx = np.iscomplexobj(a)
    for i in range(nblocks):                               # :106
        width = min(b, n - i * b)
        if max_cols is not None:
            width = min(width, max_cols - q.shape[1])
            if width <= 0:
                break
        om = omega_block(rng, n, width, cplx)              # :112-114
        y = a @ om                                         # :115
        if q.shape[1]:                                     # :116-118
            y -= q @ (q.conj().T @ y)
            y -= q @ (q.conj().T @ y)
        for _ in range(power_iters):                       # unpinned extension
            p = reduced_qr(y)[0]
            zq = reduced_qr(a.conj().T @ p)[0]
            y = a @ zq
            if q.shape[1]:
                y -= q @ (q.conj().T @ y)
                y -= q @ (q.conj().T @ y)
        p, t = reduced_qr(y)                               # :119
        keep = np.abs(np.diagonal(t)) >= trim_cut          # :120-121
        p = p[:, keep]
        if p.shape[1]:
            captured.append(sum_sq(p.conj().T @ a))        # :123
            q = np.hstack([q, p])                          # :124
        widths.append(p.shape[1])
        res2 = gf2 - math.fsum(captured)                   # :126
        history.append(math.sqrt(max(res2, 0.0)))          # :127
        iterations = i + 1
        if history[-1] < tol:                              # :129-131
            converged = True
            break
        if max_cols is not None and q.shape[1] >= max_cols:  # :132-133
            break
    return Basis(q, history, converged, iterations, widths)


def fixed_rank_basis(g, k: int, q: int, seed: int) -> Basis:
    """The BASELINE configs' mode: one block of width k (blocksize=k,
    max_cols=k, tol=1e-300, trim_tol=0, as test_bounds.py:71-74 builds it)
    followed by q power iterations; also returns B = Q^T G."""
    res = extract_basis(g, tol=1e-300, blocksize=k, seed=seed, max_cols=k, trim_tol=0.0,
                        power_iters=q)
    res.b = res.q.conj().T @ np.asarray(g)
    return res


# --------------------------------------------------------------- engine.py
def classify_spectrum(alphas, betas, classify_tol=1e-10):
    """engine.py:164-186 (snaps in place)."""
    a, b = alphas, betas
    n = a.size
    r = int(np.count_nonzero(b < classify_tol))
    za = int(np.count_nonzero(a < classify_tol))
    s = n - r - za
    if s < 0:
        raise ValueError("overlapping zero classifications")
    b[:r] = 0.0
    a[:r] = 1.0
    if za:
        a[n - za:] = 0.0
        b[n - za:] = 1.0
    return r, s


def spectrum_from_l_blocks(l1, l2, n, classify_tol=1e-10):
    """Default merged completion, engine.py:189-225."""
    a_raw = np.zeros(n)
    v1 = singular_values(l1)
    a_raw[: v1.size] = np.clip(v1, 0.0, 1.0)
    b_raw = np.zeros(n)
    v2 = singular_values(l2)
    if v2.size:
        b_raw[n - v2.size:] = np.clip(v2, 0.0, 1.0)[::-1]
    small_a = a_raw <= b_raw
    alphas = np.where(small_a, a_raw, np.sqrt(1.0 - b_raw**2))
    betas = np.where(small_a, np.sqrt(1.0 - a_raw**2), b_raw)
    r, s = classify_spectrum(alphas, betas, classify_tol)
    return alphas, betas, r, s, v1, v2


@dataclass
class PipelineOut:
    basis1: Basis | None
    basis2: Basis | None
    l1_block: np.ndarray
    l2_block: np.ndarray
    r_tilde: np.ndarray
    alphas: np.ndarray
    betas: np.ndarray
    r: int
    s: int
    sv1: np.ndarray
    sv2: np.ndarray


def run_pipeline(g1, g2, *, k=None, q=0, seed=0, tol=None, blocksize=100, max_cols=None,
                 trim_tol=1e-12, classify_tol=1e-10, direct=False) -> PipelineOut:
    """engine._run_pipeline + spectrum_from_l_blocks (engine.py:245-275):
    G1 uses ``seed``, G2 ``seed + 1`` (engine.py:252-253). With ``k`` set,
    both bases are fixed-rank (see fixed_rank_basis)."""
    if direct:
        c1, c2, b1, b2 = g1, g2, None, None
    else:
        if k is not None:
            b1 = fixed_rank_basis(g1, k, q, seed)
            b2 = fixed_rank_basis(g2, k, q, seed + 1)
        else:
            b1 = extract_basis(g1, tol, blocksize, seed, max_cols, trim_tol, q)
            b2 = extract_basis(g2, tol, blocksize, seed + 1, max_cols, trim_tol, q)
        c1 = b1.q.conj().T @ g1                            # engine.py:255
        c2 = b2.q.conj().T @ g2                            # engine.py:256
        b1.b, b2.b = c1, c2
    qf, rt = reduced_qr(np.vstack([c1, c2]))               # engine.py:257
    l1 = c1.shape[0]
    n = g1.shape[1]
    al, be, r, s, v1, v2 = spectrum_from_l_blocks(qf[:l1], qf[l1:], n, classify_tol)
    return PipelineOut(b1, b2, qf[:l1], qf[l1:], rt, al, be, r, s, v1, v2)


# ------------------------------------------------------------- analysis.py
def comparative(alphas, betas, r):
    """rho, theta, P1, P2, D1, D2 (analysis.py:37-79)."""
    n = alphas.size
    rho = np.full(n, np.inf)                               # :39-42
    rho[r:] = alphas[r:] / betas[r:]
    theta = np.arctan2(alphas, betas) - QUARTER_PI         # :51
    sa = float(np.sum(alphas**2))                          # :56-60
    sb = float(np.sum(betas**2))
    if sa <= 0 or sb <= 0:
        raise ValueError("degenerate spectrum")
    p1, p2 = alphas**2 / sa, betas**2 / sb
    return rho, theta, p1, p2, shannon_entropy(p1), shannon_entropy(p2)


def shannon_entropy(p) -> float:
    """analysis.py:63-79."""
    v = np.asarray(p, dtype=np.float64)
    nz = v[v > 0]
    d = -float(np.sum(nz * np.log(nz))) / math.log(v.size)
    return min(max(d, 0.0), 1.0) + 0.0


# ------------------------------------------------------ stage-level checks
def principal_angles_max(qa: np.ndarray, qb: np.ndarray) -> float:
    """Largest principal angle (radians) between span(qa) and span(qb),
    both with orthonormal columns; sine-based for accuracy at small angles."""
    if qa.shape[1] == 0:
        return 0.0
    proj = qb - qa @ (qa.conj().T @ qb)
    s = np.linalg.svd(proj, compute_uv=False)
    return float(np.arcsin(min(1.0, s.max()))) if s.size else 0.0
