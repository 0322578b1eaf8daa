"""fp32-resident pairs (the cfg4 family): G stays float32 in HBM and every
GEMM pass promotes row chunks to fp64 (rgsv_convert_f32), which is exactly
the reference's up-front promotion (core.py:51-54). Results must match the
oracle on the promoted data at the fp64 parity tolerances."""

import numpy as np
import pytest
import torch

from oracle import rgsv_oracle as orc
from paper_2404_09459_b200.workloads import CONFIGS, make_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg():
    import paper_2404_09459_b200 as rg

    rg._native.require_device()
    return rg


def _f32_pair(m=3000, p=2400, n=300):
    cfg = CONFIGS["cfg4"]
    g1, g2 = make_pair(cfg, data_seed=11, m=m, p=p, n=n)
    return g1.astype(np.float32), g2.astype(np.float32)


def test_convert_f32_exact(rg):
    a = np.random.default_rng(0).standard_normal((37, 29)).astype(np.float32)
    t = torch.from_numpy(a).cuda()
    dm = rg.device.to_device(t, "a", keep_f32=True)
    out = [c.t.cpu().numpy() for _, _, c in rg.device.f64_chunks(dm, rows=10)]
    assert np.array_equal(np.vstack(out), a.astype(np.float64))


@pytest.mark.parametrize("chunk_rows", [None, 701])
def test_chunked_chain_matches_oracle(rg, chunk_rows):
    g1, _ = _f32_pair()
    k, q, seed, s = 24, 1, 3, CONFIGS["cfg4"].s
    dm = rg.device.to_device(torch.from_numpy(g1).cuda(), "g", keep_f32=True)
    qm, b, hist = rg.rangefinder.chunked_chain(dm, k, q, seed, chunk_rows=chunk_rows)
    g64 = g1.astype(np.float64)
    o = orc.fixed_rank_basis(g64, k, q, seed)
    ho = o.residual_history
    assert abs(hist[0] - ho[0]) <= 1e-13 * ho[0]
    e, eo = hist[0] ** 2 - hist[1] ** 2, ho[0] ** 2 - ho[1] ** 2
    assert abs(e - eo) <= 1e-12 * eo
    bh = b.cpu().numpy()[:k, : g1.shape[1]]
    ss = min(s, k) // 2  # leading signal rows (well separated)
    assert np.linalg.norm(bh[:ss] - o.b[:ss]) <= 1e-12 * np.linalg.norm(o.b[:ss])
    qh = qm.cpu().numpy()[:, :k]
    assert np.linalg.norm(qh.T @ qh - np.eye(k)) <= 1e-12 * np.sqrt(k)


def test_f32_pair_compare_matches_f64(rg):
    g1, g2 = _f32_pair()
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(24, 5, 1), f32_mode="promote")
    r32 = rg.compare(rg.GmpPair(g1, g2), opts)
    r64 = rg.compare(rg.GmpPair(g1.astype(np.float64), g2.astype(np.float64)), opts)
    assert np.array_equal(r32.spectrum.alphas, r64.spectrum.alphas)
    assert (r32.spectrum.r, r32.spectrum.s) == (r64.spectrum.r, r64.spectrum.s)
    assert np.max(np.abs(r32.theta - r64.theta)) <= 1e-12
    assert abs(r32.d1 - r64.d1) <= 1e-12 and abs(r32.d2 - r64.d2) <= 1e-12
    o = orc.run_pipeline(g1.astype(np.float64), g2.astype(np.float64), k=24, q=1, seed=5)
    assert np.array_equal(r32.spectrum.alphas, o.alphas)


def test_wide_stacked_small_gsvd_l576(rg):
    """Stacked width l = 576 > 512 (cfg4's 2k): chol/CholQR3 wide branch."""
    rng = np.random.default_rng(1)
    n, k = 1200, 288
    b1 = rng.standard_normal((k, n))
    b2 = rng.standard_normal((k, n))
    t1 = torch.from_numpy(b1).cuda()
    t2 = torch.from_numpy(b2).cuda()
    out = rg.device.small_spectrum(t1, k, t2, k, n, 1e-10)
    qf, _ = orc.reduced_qr(np.vstack([b1, b2]))
    sv1 = np.linalg.svd(qf[:k], compute_uv=False)
    sv2 = np.linalg.svd(qf[k:], compute_uv=False)
    assert np.max(np.abs(out["sv1"] - sv1)) <= 1e-12
    assert np.max(np.abs(out["sv2"] - sv2)) <= 1e-12
    al, be, r, s, *_ = orc.spectrum_from_l_blocks(qf[:k], qf[k:], n, 1e-10)
    assert out["counts"] == (r, s)
    assert np.max(np.abs(out["alphas"] - al)) <= 1e-12
