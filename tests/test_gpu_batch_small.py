"""Batched small-pair path (rgsv_batch_gsvd, SURVEY.md §8 cfg3 shapes).

Each pair of a batch must equal the single-pair device pipeline and the
oracle's fixed-rank restatement on the same seeds: spectrum and counts
exactly, residual energies to 1e-12, the leading s rows of B to 1e-12
(parity contract), comparative quantities to 1e-12.
"""

import numpy as np
import pytest
import torch

from oracle import rgsv_oracle as orc
from paper_2404_09459_b200.workloads import CONFIGS, batch_seeds, make_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg():
    import paper_2404_09459_b200 as rg

    rg._native.require_device()
    return rg


def _pairs(rg, cfg, B, m=None, p=None):
    hosts, pairs, seeds = [], [], []
    for j in range(B):
        ds, os_ = batch_seeds(j)
        g1, g2 = make_pair(cfg, data_seed=ds, m=m, p=p)
        hosts.append((g1, g2))
        pairs.append(rg.GmpPair.resident(torch.from_numpy(g1).cuda(),
                                         torch.from_numpy(g2).cuda()))
        seeds.append(os_)
    return hosts, pairs, seeds


@pytest.mark.parametrize("B,m,p", [(6, None, None), (3, 1000, 517), (2, 9000, 77),
                                   (2, 12000, 77)])
def test_batch_matches_single_and_oracle(rg, B, m, p):
    cfg = CONFIGS["cfg3"]
    hosts, pairs, seeds = _pairs(rg, cfg, B, m, p)
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))
    # 12000 rows exceed the clustered Y slice (8-CTA clusters hold ~9200):
    # the engine takes the per-pair stream plan instead, and the results must
    # not depend on which path ran
    assert rg.device.small_batch_fits(max(hosts[0][0].shape[0], hosts[0][1].shape[0]), cfg.n,
                                      cfg.k, cfg.k) == (m != 12000)
    runs = rg.engine.run_device_batch(pairs, opts, seeds)
    for j, (run, (g1, g2)) in enumerate(zip(runs, hosts)):
        single = rg.engine.run_device_pipeline(
            pairs[j], rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, seeds[j],
                                                                               cfg.q)))
        assert np.array_equal(run.alphas, single.alphas)
        assert (run.r, run.s) == (single.r, single.s)
        for a, b in ((run.theta, single.theta), (run.p1, single.p1), (run.p2, single.p2)):
            assert np.max(np.abs(a - b)) <= 1e-12
        o = orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=seeds[j])
        assert np.array_equal(run.alphas, o.alphas) and (run.r, run.s) == (o.r, o.s)
        for basis, ob in ((run.basis1, o.basis1), (run.basis2, o.basis2)):
            h, ho = basis.residual_history, ob.residual_history
            assert abs(h[0] - ho[0]) <= 1e-13 * ho[0]
            e, eo = h[0] ** 2 - h[1] ** 2, ho[0] ** 2 - ho[1] ** 2
            assert abs(e - eo) <= 1e-12 * eo


@pytest.mark.parametrize("n,k,q,m,p", [(50, 12, 1, 1003, 700),    # <64,16>: ragged columns (n < 64)
                                       (63, 16, 2, 2500, 1900),   # odd n, two power iterations
                                       (64, 16, 0, 2001, 1333),   # q = 0, partial last blocks
                                       (100, 16, 1, 1500, 900),   # <128,16> ring instantiation
                                       (128, 16, 1, 900, 1100),   # <128,16>, full width
                                       (40, 20, 1, 600, 450)])    # <64,32>
def test_batch_other_shapes_match_single_and_oracle(rg, n, k, q, m, p):
    """Every kernel instantiation behind rgsv_batch_gsvd (register-streamed
    <64,16> incl. its predicated loads for n < 64 and partial row blocks, and
    the ring-staged <64,32> and <128,16>) against the single-pair
    pipeline and the oracle, on ill-conditioned cfg3-structured pairs."""
    import dataclasses

    cfg = dataclasses.replace(CONFIGS["cfg3"], n=n, k=k, q=q, s=min(8, k // 2), shared=min(4, k // 4))
    hosts, pairs, seeds = _pairs(rg, cfg, 3, m, p)
    assert rg.device.small_batch_fits(max(m, p), n, k, k)
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(k, 0, q))
    runs = rg.engine.run_device_batch(pairs, opts, seeds)
    for j, (run, (g1, g2)) in enumerate(zip(runs, hosts)):
        o = orc.run_pipeline(g1, g2, k=k, q=q, seed=seeds[j])
        assert np.array_equal(run.alphas, o.alphas) and (run.r, run.s) == (o.r, o.s)
        for basis, ob in ((run.basis1, o.basis1), (run.basis2, o.basis2)):
            h, ho = basis.residual_history, ob.residual_history
            assert abs(h[0] - ho[0]) <= 1e-13 * ho[0]
            e, eo = h[0] ** 2 - h[1] ** 2, ho[0] ** 2 - ho[1] ** 2
            assert abs(e - eo) <= 1e-12 * eo
        single = rg.engine.run_device_pipeline(
            pairs[j], rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(k, seeds[j], q)))
        assert np.array_equal(run.alphas, single.alphas)
        for a, b in ((run.theta, single.theta), (run.p1, single.p1), (run.p2, single.p2)):
            assert np.max(np.abs(a - b)) <= 1e-12


def test_batch_projections_match_oracle_rows(rg):
    cfg = CONFIGS["cfg3"]
    B = 4
    hosts, pairs, seeds = _pairs(rg, cfg, B)
    plan = rg.device.small_batch_plan(B, cfg.n, cfg.k)
    plan.set_pairs([(pr.g1, pr.g2) for pr in pairs])
    plan.set_seeds(seeds)
    kp, ldo = 16, 64
    bo = torch.zeros((2 * B, kp, ldo), dtype=torch.float64, device="cuda")
    plan.launch(cfg.q, 1e-10, b_out=bo)
    plan.fetch()
    b = bo.cpu().numpy()
    s = cfg.s
    for j, (g1, g2) in enumerate(hosts):
        for i, (g, sd) in enumerate(((g1, seeds[j]), (g2, seeds[j] + 1))):
            ob = orc.fixed_rank_basis(g, cfg.k, cfg.q, sd).b
            lead = ob[:s]
            assert np.linalg.norm(b[2 * j + i, :s, : cfg.n] - lead) <= 1e-12 * np.linalg.norm(lead)
            # full k-row block: same span (rows are an orthonormal-basis image)
            sv_d = np.linalg.svd(b[2 * j + i, : cfg.k, : cfg.n], compute_uv=False)
            sv_o = np.linalg.svd(ob, compute_uv=False)
            assert np.max(np.abs(sv_d[:s] - sv_o[:s])) <= 1e-12 * sv_o[0]
            assert not np.any(b[2 * j + i, cfg.k:])


def test_batch_full_cfg3_scale_invariants(rg):
    """All 4096 cfg3 pairs in one call: size-independent properties (every
    spectrum is the F2 closed form, energies below |G|^2, entropies fixed)."""
    cfg = CONFIGS["cfg3"]
    B = cfg.batch
    rng = torch.Generator(device="cuda").manual_seed(0)
    g1 = torch.randn((B, cfg.m, cfg.n), generator=rng, device="cuda", dtype=torch.float64)
    g2 = torch.randn((B, cfg.p, cfg.n), generator=rng, device="cuda", dtype=torch.float64)
    pairs = [rg.GmpPair.resident(g1[j], g2[j]) for j in range(B)]
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))
    runs = rg.engine.run_device_batch(pairs, opts, [2 * j for j in range(B)])
    closed = np.r_[np.ones(cfg.k), np.zeros(cfg.n - cfg.k)]
    for run in runs[:: 97]:
        assert np.array_equal(run.alphas, closed) and (run.r, run.s) == (cfg.k, 0)
        h = run.basis1.residual_history
        assert 0.0 < h[1] < h[0]
    # spot-check a few pairs against the single-pair pipeline
    for j in (0, 1234, B - 1):
        single = rg.engine.run_device_pipeline(
            pairs[j], rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 2 * j, cfg.q)))
        e_b = runs[j].basis1.residual_history
        e_s = single.basis1.residual_history
        assert abs((e_b[0] ** 2 - e_b[1] ** 2) - (e_s[0] ** 2 - e_s[1] ** 2)) <= 1e-12 * e_s[0] ** 2


def test_host_stream_batch_equals_resident(rg):
    """compare_batch on host (g1, g2) arrays (streamed, copy/compute overlap)
    returns exactly what the resident-pair batch returns."""
    cfg = CONFIGS["cfg0"]
    hosts = [make_pair(cfg, data_seed=40 + j) for j in range(3)]
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))
    seeds = [5, 6, 7]
    res_dev = rg.compare_batch([rg.GmpPair.resident(torch.from_numpy(a).cuda(),
                                                    torch.from_numpy(b).cuda())
                                for a, b in hosts], opts, seeds)
    pinned = [(torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory())
              for a, b in hosts]
    for _ in range(3):  # eager, capture, replay
        res_host = rg.compare_batch(pinned, opts, seeds)
        for x, y in zip(res_dev, res_host):
            assert np.array_equal(x.spectrum.alphas, y.spectrum.alphas)
            assert np.array_equal(x.theta, y.theta) and x.d1 == y.d1 and x.d2 == y.d2
    # numpy (pageable) inputs work too
    res_np = rg.compare_batch(hosts, opts, seeds)
    assert np.array_equal(res_np[2].p1, res_dev[2].p1)
    bad = [(hosts[0][0].copy(), hosts[0][1])]
    bad[0][0][3, 4] = np.nan
    with pytest.raises(rg.ValidationError):
        rg.compare_batch(bad, opts, [0])


def test_batch_results_survive_later_calls_and_flag_bad_input(rg):
    """Each compare_batch call returns views of its OWN pinned result
    buffers: a second call (new seeds, new pair set) leaves the first
    call's reports untouched. The device-side status word carries the
    finiteness and GsvSpectrum checks: a NaN in one pair's G raises
    ValidationError; a shape mismatch raises DimensionError."""
    cfg = CONFIGS["cfg3"]
    hosts, pairs, seeds = _pairs(rg, cfg, 4, m=900, p=700)
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))
    first = rg.compare_batch(pairs, opts, seeds)
    keep = [(r.theta.copy(), r.d1, r.spectrum.alphas.copy()) for r in first]
    second = rg.compare_batch(pairs[::-1], opts, [s + 100 for s in seeds])
    assert len(second) == 4
    for r, (th, d1, al) in zip(first, keep):
        assert np.array_equal(r.theta, th) and r.d1 == d1 and np.array_equal(r.spectrum.alphas, al)
    for j, (g1, g2) in enumerate(hosts):  # both calls still match the oracle
        o = orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=seeds[j])
        assert np.array_equal(first[j].spectrum.alphas, o.alphas)
        o2 = orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=seeds[j] + 100)
        assert np.array_equal(second[3 - j].spectrum.alphas, o2.alphas)
        assert abs(second[3 - j].d2 - orc.comparative(o2.alphas, o2.betas, o2.r)[5]) <= 1e-12
    bad_g = pairs[2].g1.t.clone()
    bad_g[5, 7] = float("nan")
    bad = list(pairs)
    bad[2] = rg.GmpPair.resident(bad_g, pairs[2].g2.t)
    with pytest.raises(rg.ValidationError):
        rg.compare_batch(bad, opts, seeds)
    odd = list(pairs)
    odd[1] = rg.GmpPair.resident(pairs[1].g1.t[:800], pairs[1].g2.t)
    with pytest.raises(rg.DimensionError):
        rg.compare_batch(odd, opts, seeds)
