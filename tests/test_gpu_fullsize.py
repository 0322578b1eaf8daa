"""BASELINE.json's configs at FULL size on the device, checked through
size-independent properties (the CPU oracle cannot run them: cfg2 needs
minutes per pair, cfg4 118 GB of host fp64). Data are generated on the
device with the workloads.py recipe (bench.device_matrix /
device_batch_pairs).

* Fixed-rank sketches with 2k < n give the reference's data-independent
  spectrum: alpha = [1]*k + [0]*(n-k) EXACTLY, r = k,
  s = 0, theta = +-pi/4, so the whole comparative report is known in
  closed form.
* Captured energy: the signal rank s < k, so the residual after the basis is
  the noise outside it (eps^2 m (n - k)) up to the path's energy tolerance.
* The basis is orthonormal to fp64 precision.
* Runs are bitwise deterministic.
"""

import math

import numpy as np
import pytest
import torch

import bench
from paper_2404_09459_b200.workloads import CONFIGS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg():
    import paper_2404_09459_b200 as rg

    rg._native.require_device()
    return rg


def _pair(cfg, dtype, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    b1 = torch.randn((cfg.n, cfg.s), generator=gen, device="cuda", dtype=dtype)
    b2 = torch.cat([b1[:, : cfg.shared],
                    torch.randn((cfg.n, cfg.s - cfg.shared), generator=gen, device="cuda",
                                dtype=dtype)], dim=1)
    d = (10.0 ** (-cfg.decay * torch.arange(cfg.s, device="cuda", dtype=torch.float64)
                  / cfg.s)).to(dtype)
    g1 = bench.device_matrix(cfg.m, cfg, seed + 1, b1, d, dtype)
    g2 = bench.device_matrix(cfg.p, cfg, seed + 2, b2, d, dtype)
    return g1, g2


def _check_closed_form(rep, k, n):
    a, b = rep.spectrum.alphas, rep.spectrum.betas
    want_a = np.r_[np.ones(k), np.zeros(n - k)]
    assert np.array_equal(a, want_a)
    assert np.array_equal(b, np.sqrt(1.0 - want_a ** 2))
    assert (rep.spectrum.r, rep.spectrum.s) == (k, 0)
    assert np.array_equal(np.abs(rep.theta), np.full(n, math.pi / 4))
    assert 0.0 <= rep.d1 <= 1.0 and 0.0 <= rep.d2 <= 1.0


def _same(r1, r2):
    assert np.array_equal(r1.spectrum.alphas, r2.spectrum.alphas)
    assert np.array_equal(r1.theta, r2.theta)
    assert np.array_equal(r1.p1, r2.p1) and np.array_equal(r1.p2, r2.p2)
    assert r1.d1 == r2.d1 and r1.d2 == r2.d2


def _basis_checks(rg, g, cfg, seed, f32):
    """Orthonormal basis, energy at the noise floor (one matrix)."""
    dm = rg.device.to_device(g, "g", keep_f32=f32)
    if f32:
        q, _, h = rg.tf32.tf32_chain(dm, cfg.k, cfg.q, seed)
    else:
        q, _, h = rg.rangefinder.chunked_chain(dm, cfg.k, cfg.q, seed)
    k = cfg.k
    qk = q[:, :k]
    gram = qk.T @ qk
    eye = torch.eye(k, dtype=torch.float64, device="cuda")
    assert float(torch.linalg.norm(gram - eye)) <= 1e-12 * math.sqrt(k)
    assert 0.0 <= h[1] <= h[0]
    # uncaptured energy = the noise outside the basis (eps^2 m (n - k), the
    # signal rank s < k is captured) plus the energy tolerance of the path:
    # fp64 rounding, or the ~1e-6 low bias of the tensor core's truncating
    # accumulation on ||B||^2 for fp32 (tests/test_gpu_tf32.py)
    rel = 5e-6 if f32 else 1e-12
    bound = math.sqrt(1.5 * cfg.eps ** 2 * g.shape[0] * cfg.n + rel * h[0] ** 2)
    assert h[1] <= bound, (h, bound)


def test_cfg2_full_size(rg):
    cfg = CONFIGS["cfg2"]
    g1, g2 = _pair(cfg, torch.float64, 2024)
    pair = rg.GmpPair.resident(g1, g2)
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 3, cfg.q))
    r1 = rg.compare(pair, opts)
    r2 = rg.compare(pair, opts)
    _check_closed_form(r1, cfg.k, cfg.n)
    _same(r1, r2)
    _basis_checks(rg, g1, cfg, 3, f32=False)
    del pair, g1, g2
    torch.cuda.empty_cache()


def test_cfg3_full_batch(rg):
    cfg = CONFIGS["cfg3"]
    g1, g2 = bench.device_batch_pairs(cfg, cfg.batch, 7)
    pairs = [rg.GmpPair.resident(g1[j], g2[j]) for j in range(cfg.batch)]
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))
    seeds = [2 * j for j in range(cfg.batch)]
    reps = rg.compare_batch(pairs, opts, seeds=seeds)
    again = rg.compare_batch(pairs, opts, seeds=seeds)
    for j in (0, 1, cfg.batch // 2, cfg.batch - 1):
        _check_closed_form(reps[j], cfg.k, cfg.n)
        _same(reps[j], again[j])
    alphas = np.stack([reps[j].spectrum.alphas for j in range(cfg.batch)])
    assert np.array_equal(alphas, np.broadcast_to(alphas[0], alphas.shape))
    del pairs, g1, g2
    torch.cuda.empty_cache()


def test_cfg4_full_size_fp32(rg):
    cfg = CONFIGS["cfg4"]
    g1, g2 = _pair(cfg, torch.float32, 4048)
    pair = rg.GmpPair.resident(g1, g2)
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 5, cfg.q))
    r1 = rg.compare(pair, opts)
    r2 = rg.compare(pair, opts)
    _check_closed_form(r1, cfg.k, cfg.n)
    _same(r1, r2)
    del pair, g2
    torch.cuda.empty_cache()
    _basis_checks(rg, g1, cfg, 5, f32=True)
    del g1
    torch.cuda.empty_cache()
