"""Stage-level oracle parity at the BASELINE shapes, and the timed replay
path with CHANGED seeds.

* cfg2 at full size (200000 / 150000 x 4000, k = 120, q = 2) against the
  CPU oracle on identical Omega (SURVEY.md §0 contract (ii)): captured
  energy <= 1e-13 relative, leading-s signal subspace angle <= 1e-12, rows
  0..s-1 of B <= 1e-12 relative, ||Q^T Q - I||_F <= 1e-12 sqrt(k), full
  k-span angle <= 1e-6 (condition-scaled, F3), spectrum equal.
* cfg4's column shape (n = 8192, k = 288, q = 1) on a 1/50-row instance
  (m = 20000, p = 16000) through the DEFAULT fp32 path (tf32x3 tensor-core
  chain) against the fp64 oracle on the promoted data: GSVs and theta
  <= 1e-4 (BASELINE.json's cfg4 tolerance), captured energy <= 5e-6.
* Replay: the bench replays captured CUDA graphs with new Omega seeds every
  step. A graph captured at seed s and replayed at s' must match the oracle
  at s' (and differ from s), for PairPlan, BatchPlan and SmallBatchPlan.
  The F2 spectrum is Omega-independent, so the checks are on the bases and
  energies.
"""

import math

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


def _opts(rg, k, q, seed):
    return rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(k, seed, q))


def _sin_angle(qa, qb):
    """Sine of the largest principal angle between span(qa) and span(qb)
    (orthonormal columns)."""
    return orc.principal_angles_max(qa, qb)


def _stage_checks(g, q, ob, s_sig, *, energy_tol, lead_tol, full_tol, brow_tol):
    k = ob.q.shape[1]
    assert np.linalg.norm(q.T @ q - np.eye(k)) <= 1e-12 * math.sqrt(k)
    assert _sin_angle(ob.q[:, :s_sig], q[:, :s_sig]) <= lead_tol
    assert _sin_angle(ob.q, q) <= full_tol
    b = q.T @ g
    e_ref = orc.sum_sq(ob.b)
    assert abs(orc.sum_sq(b) - e_ref) <= energy_tol * e_ref
    bref = ob.b
    assert np.linalg.norm(b[:s_sig] - bref[:s_sig]) <= brow_tol * np.linalg.norm(bref[:s_sig])


def test_cfg2_full_size_stage_parity(rg):
    cfg = CONFIGS["cfg2"]
    g1, g2 = make_pair(cfg)
    seed = 11
    pair = rg.GmpPair(g1, g2, check_rank=False)
    run = rg.engine.run_device_pipeline(pair, _opts(rg, cfg.k, cfg.q, seed))
    o = orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=seed)
    assert np.array_equal(run.alphas, o.alphas) and (run.r, run.s) == (o.r, o.s)
    _, theta, p1, p2, d1, d2 = orc.comparative(o.alphas, o.betas, o.r)
    assert np.max(np.abs(run.theta - theta)) <= 1e-15
    assert abs(run.d1 - d1) <= 1e-14 and abs(run.d2 - d2) <= 1e-14
    plan = run.plan
    for g, sub, bres, ob in ((g1, plan.s1, run.basis1, o.basis1),
                             (g2, plan.s2, run.basis2, o.basis2)):
        q = sub.q[:, : cfg.k].cpu().numpy()
        # ||G||_F (fused into the sketch GEMM) and the captured energy of
        # the pipeline's own residual history
        h = bres.residual_history
        assert abs(h[0] - ob.residual_history[0]) <= 1e-14 * ob.residual_history[0]
        e_ref = orc.sum_sq(ob.b)
        assert abs(h[0] ** 2 - h[1] ** 2 - e_ref) <= 1e-12 * e_ref
        _stage_checks(g, q, ob, cfg.s, energy_tol=1e-13, lead_tol=1e-12, full_tol=1e-6,
                      brow_tol=1e-12)
        bdev = sub.b[: cfg.k, : cfg.n].cpu().numpy()
        bref = ob.b
        assert np.linalg.norm(bdev[: cfg.s] - bref[: cfg.s]) <= 1e-12 * np.linalg.norm(bref[: cfg.s])
    del pair, run
    torch.cuda.empty_cache()


def test_cfg4_columns_instance_vs_oracle(rg):
    """n = 8192, k = 288 (cfg4's real column shape) on 1/50 of the rows,
    fp32 through the default tf32x3 tensor-core chain."""
    cfg = CONFIGS["cfg4"]
    m, p = cfg.m // 50, cfg.p // 50
    g1, g2 = make_pair(cfg, data_seed=5, m=m, p=p)
    f1, f2 = g1.astype(np.float32), g2.astype(np.float32)
    del g1, g2
    seed = 9
    pair = rg.GmpPair(f1, f2, check_rank=False)
    rep = rg.compare(pair, _opts(rg, cfg.k, cfg.q, seed))
    h1, h2 = f1.astype(np.float64), f2.astype(np.float64)
    o = orc.run_pipeline(h1, h2, k=cfg.k, q=cfg.q, seed=seed)
    assert np.max(np.abs(rep.spectrum.alphas - o.alphas)) <= 1e-4
    assert np.max(np.abs(rep.spectrum.betas - o.betas)) <= 1e-4
    assert (rep.spectrum.r, rep.spectrum.s) == (o.r, o.s)
    _, theta, _, _, d1, d2 = orc.comparative(o.alphas, o.betas, o.r)
    assert np.max(np.abs(rep.theta - theta)) <= 1e-4
    assert abs(rep.d1 - d1) <= 1e-4 and abs(rep.d2 - d2) <= 1e-4
    # stage level on G1 through the same chain the pair ran
    dm = rg.device.to_device(torch.from_numpy(f1).cuda(), "g", keep_f32=True)
    qm, b, hist = rg.tf32.tf32_chain(dm, cfg.k, cfg.q, seed)
    ob = o.basis1
    ho = ob.residual_history
    assert abs(hist[0] - ho[0]) <= 1e-13 * ho[0]
    e, eo = hist[0] ** 2 - hist[1] ** 2, orc.sum_sq(ob.b)
    assert abs(e - eo) <= 5e-6 * eo, (e, eo)
    q = qm[:, : cfg.k].cpu().numpy()
    assert np.linalg.norm(q.T @ q - np.eye(cfg.k)) <= 1e-12 * math.sqrt(cfg.k)
    lead = cfg.s // 2  # leading signal directions (well separated from the noise)
    assert _sin_angle(ob.q[:, :lead], q[:, :lead]) <= 1e-4
    bh = b[: cfg.k, : cfg.n].cpu().numpy()
    assert np.linalg.norm(bh[:lead] - ob.b[:lead]) <= 1e-4 * np.linalg.norm(ob.b[:lead])
    del pair, dm, qm, b
    torch.cuda.empty_cache()


def _energy(bres):
    h = bres.residual_history
    return h[0] ** 2 - h[1] ** 2


def test_pair_graph_replay_with_new_seed(rg):
    """PairPlan: eager at s, captured on the second sighting, replayed at s'."""
    cfg = CONFIGS["cfg0"]  # s = 20 < k: k - s noise directions that follow Omega
    g1, g2 = make_pair(cfg, data_seed=21, m=6000, p=5000, n=600)
    pair = rg.GmpPair(g1, g2, check_rank=False)
    k, q = 40, 2
    s0, s1 = 3, 77
    replays0 = rg.device.GRAPH_REPLAYS[0]
    for _ in range(2):  # eager, then capture (+ first replay)
        rg.engine.run_device_pipeline(pair, _opts(rg, k, q, s0))
    run = rg.engine.run_device_pipeline(pair, _opts(rg, k, q, s1))  # replay, new seed
    assert rg.device.GRAPH_REPLAYS[0] >= replays0 + 2, "the timed path must replay the graph"
    for g, sub, bres, seed in ((g1, run.plan.s1, run.basis1, s1),
                               (g2, run.plan.s2, run.basis2, s1 + 1)):
        ob = orc.fixed_rank_basis(g, k, q, seed)
        old = orc.fixed_rank_basis(g, k, q, s0 if seed == s1 else s0 + 1)
        qd = sub.q[:, :k].cpu().numpy()
        _stage_checks(g, qd, ob, cfg.s, energy_tol=1e-13, lead_tol=1e-12, full_tol=1e-6,
                      brow_tol=1e-12)
        # the noise directions of the basis follow the seed: the stale
        # seed's basis is far away, the new one is not
        assert _sin_angle(old.q, qd) > 1e-3
        assert abs(_energy(bres) - orc.sum_sq(ob.b)) <= 1e-12 * orc.sum_sq(ob.b)


def test_batch_graph_replay_with_new_seeds(rg):
    """BatchPlan (compare_batch on resident pairs, one graph for all)."""
    cfg = CONFIGS["cfg0"]
    hosts = [make_pair(cfg, data_seed=d, m=900, p=700) for d in (31, 32, 33)]
    pairs = [rg.GmpPair(a, b, check_rank=False) for a, b in hosts]
    opts = _opts(rg, cfg.k, cfg.q, 0)
    for _ in range(3):  # eager, capture, replay
        rg.engine.run_device_batch(pairs, opts, seeds=[1, 2, 3])
    new = [40, 50, 60]
    runs = rg.engine.run_device_batch(pairs, opts, seeds=new)
    for (g1, g2), run, sd in zip(hosts, runs, new):
        for g, sub, bres, seed in ((g1, run.plan.s1, run.basis1, sd),
                                   (g2, run.plan.s2, run.basis2, sd + 1)):
            ob = orc.fixed_rank_basis(g, cfg.k, cfg.q, seed)
            qd = sub.q[:, : cfg.k].cpu().numpy()
            _stage_checks(g, qd, ob, cfg.s, energy_tol=1e-13, lead_tol=1e-12, full_tol=1e-6,
                          brow_tol=1e-12)
            assert abs(_energy(bres) - orc.sum_sq(ob.b)) <= 1e-12 * orc.sum_sq(ob.b)


def test_small_batch_new_seeds(rg):
    """SmallBatchPlan (cfg3 kernels): a second call with other seeds."""
    cfg = CONFIGS["cfg3"]
    hosts = [make_pair(cfg, data_seed=j, m=1200, p=900) for j in range(6)]
    pairs = [rg.GmpPair.resident(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
             for a, b in hosts]
    opts = _opts(rg, cfg.k, cfg.q, 0)
    rg.engine.run_device_batch(pairs, opts, seeds=[2 * j for j in range(6)])
    new = [1000 + 2 * j for j in range(6)]
    runs = rg.engine.run_device_batch(pairs, opts, seeds=new)
    for j in (0, 3, 5):
        g1, g2 = hosts[j]
        for g, bres, seed in ((g1, runs[j].basis1, new[j]), (g2, runs[j].basis2, new[j] + 1)):
            e_ref = orc.sum_sq(orc.fixed_rank_basis(g, cfg.k, cfg.q, seed).b)
            assert abs(_energy(bres) - e_ref) <= 1e-12 * e_ref
