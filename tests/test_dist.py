"""Row-sharded multi-rank pipeline (paper_2404_09459_b200/dist.py and the
native rgsv_sketch_project_sharded).

CPU (gloo, world_size 2): the sharded algorithm -- which partials are
summed where, the CholeskyQR shift from the GLOBAL row count, the wide QR
of the replicated Z -- restated on torch-CPU below (`sharded_chain_cpu`,
the specification rgsv_sketch_project_sharded implements, capi.cu) with
every cross-rank sum going through the product's ``dist.Comm`` in its
torch mode; checked against the oracle. Plus ``Comm``'s host collectives.

GPU: the NATIVE chain with two processes on one GPU over gloo (the host
all-reduce hook, Comm mode "torch"), fp64 and fp32 shards, against the
oracle; and a 1-rank NCCL communicator owned by librgsv (Comm mode "nccl")
through eager, captured and replayed CUDA graphs with changing seeds.
Several ranks on one GPU cannot use NCCL (duplicate device) and must not
run kernels that wait on each other, hence gloo for the multi-rank case.
"""

import math
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rgsv_oracle as orc
from paper_2404_09459_b200 import dist as rdist
from paper_2404_09459_b200.workloads import CONFIGS, make_pair


# ------------------------------------------------ CPU restatement (test only)
def _chol_linv(gram, k, kp, shift_rows):
    a = gram[:k, :k].clone()
    if shift_rows > 0:  # shifted CholeskyQR (Fukaya et al.), cholqr.cu k_chol_*
        tr = float(torch.trace(a))
        a += 11.0 * (shift_rows * k + k * (k + 1)) * 2.0 ** -53 * tr * torch.eye(k, dtype=a.dtype)
    linv = torch.eye(kp, dtype=torch.float64)
    linv[:k, :k] = torch.linalg.inv(torch.linalg.cholesky(a))
    return linv


def _tall_cholqr3(comm, y, m_total, k, kp):
    for step in range(3):
        gram = comm.allreduce_tensor(y.T @ y)
        y = y @ _chol_linv(gram, k, kp, m_total if step == 0 else 0).T
    return y


def _wide_cholqr3(zt, n, k, kp):
    for step in range(3):
        gram = zt @ zt.T
        zt = _chol_linv(gram, k, kp, n if step == 0 else 0) @ zt
    return zt


def sharded_chain_cpu(comm, g_local, m_total, n, k, q, seed):
    """rgsv_sketch_project_sharded's schedule on torch-CPU."""
    kp = (k + 15) // 16 * 16
    om = torch.zeros((n, kp), dtype=torch.float64)
    om[:, :k] = torch.from_numpy(orc.gaussian_matrix(n, k, seed))
    ss = comm.allreduce_tensor(torch.tensor([float((g_local ** 2).sum())], dtype=torch.float64))
    qb = _tall_cholqr3(comm, g_local @ om, m_total, k, kp)
    for _ in range(q):
        zt = comm.allreduce_tensor(qb.T @ g_local)
        qht = _wide_cholqr3(zt, n, k, kp)
        qb = _tall_cholqr3(comm, g_local @ qht.T, m_total, k, kp)
    b = comm.allreduce_tensor(qb.T @ g_local)
    return b, float(ss[0]), float((b ** 2).sum())


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _cpu_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = rdist.Comm()  # auto: gloo with 2 ranks -> host collectives
    assert comm.mode == "torch" and comm.world == world and comm.rank == rank
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg, m=700, p=500)
    out = {}
    for name, g, seed in (("1", g1, 3), ("2", g2, 4)):
        r0, r1 = rdist.shard_rows(g.shape[0], rank, world)
        b, gf2, e = sharded_chain_cpu(comm, torch.from_numpy(g[r0:r1].copy()), g.shape[0],
                                      g.shape[1], cfg.k, cfg.q, seed)
        out["b" + name] = b.numpy()
        out["h" + name] = np.array([math.sqrt(gf2), math.sqrt(max(gf2 - e, 0.0))])
    pk = torch.arange(10, dtype=torch.float64) * (rank + 1)
    comm.broadcast(pk, 0)
    out["bcast"] = pk.numpy()
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), **out)
    dist.destroy_process_group()


def test_shard_rows_cover():
    for m in (1, 7, 20000, 200000):
        for w in (1, 2, 3, 8):
            blocks = [rdist.shard_rows(m, r, w) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in blocks) - min(b - a for a, b in blocks) <= 1


def test_comm_single_rank_without_process_group():
    comm = rdist.Comm()
    assert comm.mode == "single" and comm.world == 1
    t = torch.ones(3, dtype=torch.float64)
    assert comm.allreduce_tensor(t) is t and float(t.sum()) == 3.0
    with pytest.raises(rdist.ValidationError):
        rdist.Comm("nccl")


def test_two_rank_gloo_sharded_algorithm_matches_oracle():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_cpu_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        r0 = np.load(os.path.join(d, "r0.npz"))
        r1 = np.load(os.path.join(d, "r1.npz"))
        for key in ("b1", "b2", "h1", "h2", "bcast"):
            assert np.array_equal(r0[key], r1[key]), key  # replicated results agree
        assert np.array_equal(r0["bcast"], np.arange(10.0))  # rank 0's buffer everywhere
        cfg = CONFIGS["cfg0"]
        g1, g2 = make_pair(cfg, m=700, p=500)
        o = orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=3)
        for key, ob in (("1", o.basis1), ("2", o.basis2)):
            h = r0["h" + key]
            e_ref = orc.sum_sq(ob.b)
            assert abs(h[0] - ob.residual_history[0]) <= 1e-13 * h[0]
            assert abs(h[0] ** 2 - h[1] ** 2 - e_ref) <= 1e-12 * e_ref
            b = r0["b" + key][: cfg.k]
            s = cfg.s  # leading signal rows (same positive-R phase convention)
            assert np.linalg.norm(b[:s] - ob.b[:s]) <= 1e-11 * np.linalg.norm(ob.b[:s])
        # the spectrum from the replicated B blocks
        from oracle.rgsv_oracle import reduced_qr, spectrum_from_l_blocks

        st = np.vstack([r0["b1"][: cfg.k], r0["b2"][: cfg.k]])
        qf, _ = reduced_qr(st)
        al, _, r, s_, _, _ = spectrum_from_l_blocks(qf[: cfg.k], qf[cfg.k:], g1.shape[1])
        assert np.array_equal(al, o.alphas) and (r, s_) == (o.r, o.s)


# ---------------------------------------------------------------- GPU
def _gpu_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = rdist.Comm()
    assert comm.mode == "torch"
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg, m=3000, p=2400, n=300)
    out = {}
    r0, r1 = rdist.shard_rows(g1.shape[0], rank, world)
    s0, s1 = rdist.shard_rows(g2.shape[0], rank, world)
    for tag, dt in (("f64", torch.float64), ("f32", torch.float32)):
        a = torch.from_numpy(g1[r0:r1].copy()).to("cuda", dt)
        b = torch.from_numpy(g2[s0:s1].copy()).to("cuda", dt)
        res = rdist.compute_gsv_sharded(a, b, g1.shape[0], g2.shape[0], g1.shape[1], cfg.k,
                                        cfg.q, seed=5, comm=comm)
        out[tag + "_alphas"] = res.alphas
        out[tag + "_rs"] = np.array([res.r, res.s])
        out[tag + "_h1"] = np.array(res.residual_history1)
        out[tag + "_h2"] = np.array(res.residual_history2)
        out[tag + "_b1"] = res.b1[: cfg.k, : g1.shape[1]].cpu().numpy()
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), **out)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_native_sharded_chain_two_gloo_ranks_matches_oracle():
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_gpu_worker, args=(2, _free_port(), d), nprocs=2, join=True,
                           start_method="spawn")
        r0 = np.load(os.path.join(d, "r0.npz"))
        r1 = np.load(os.path.join(d, "r1.npz"))
        for key in r0.files:
            assert np.array_equal(r0[key], r1[key]), key  # broadcast / replicated
        cfg = CONFIGS["cfg0"]
        g1, g2 = make_pair(cfg, m=3000, p=2400, n=300)
        o = orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=5)
        # fp64 shards: the reference's stage contract
        assert np.array_equal(r0["f64_alphas"], o.alphas)
        assert list(r0["f64_rs"]) == [o.r, o.s]
        for key, ob in (("f64_h1", o.basis1), ("f64_h2", o.basis2)):
            h = r0[key]
            e_ref = orc.sum_sq(ob.b)
            assert abs(h[0] - ob.residual_history[0]) <= 1e-14 * h[0]
            assert abs(h[0] ** 2 - h[1] ** 2 - e_ref) <= 1e-12 * e_ref
        s = cfg.s
        bref = o.basis1.b
        assert np.linalg.norm(r0["f64_b1"][:s] - bref[:s]) <= 1e-12 * np.linalg.norm(bref[:s])
        # fp32 shards (tf32x3 chain): BASELINE's fp32 tolerance
        assert np.max(np.abs(r0["f32_alphas"] - o.alphas)) <= 1e-4
        assert list(r0["f32_rs"]) == [o.r, o.s]
        h = r0["f32_h1"]
        e_ref = orc.sum_sq(o.basis1.b)
        assert abs(h[0] ** 2 - h[1] ** 2 - e_ref) <= 5e-6 * e_ref


def _nccl_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0))
    import paper_2404_09459_b200 as rg

    comm = rdist.Comm("nccl")
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg, m=3000, p=2400, n=300)
    a = torch.from_numpy(g1).cuda()
    b = torch.from_numpy(g2).cuda()
    out = {}
    r0 = rg.device.GRAPH_REPLAYS[0]
    for i, seed in enumerate((1, 1, 2, 3)):  # eager, capture, replay (new seeds)
        res = rdist.compute_gsv_sharded(a, b, g1.shape[0], g2.shape[0], g1.shape[1], cfg.k,
                                        cfg.q, seed=seed, comm=comm)
        out[f"h1_{i}"] = np.array(res.residual_history1)
        out[f"alphas_{i}"] = res.alphas
        out[f"theta_{i}"] = res.report.theta
    out["replays"] = np.array([rg.device.GRAPH_REPLAYS[0] - r0])
    out["nccl"] = np.array([rg._native.lib().rgsv_nccl_version()])
    comm.close()
    np.savez(os.path.join(out_dir, "nccl.npz"), **out)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_comm_graph_capture_single_rank():
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_nccl_worker, args=(1, _free_port(), d), nprocs=1, join=True,
                           start_method="spawn")
        r = np.load(os.path.join(d, "nccl.npz"))
        assert int(r["nccl"][0]) > 0
        assert int(r["replays"][0]) >= 3  # captured once, then replayed
        cfg = CONFIGS["cfg0"]
        g1, g2 = make_pair(cfg, m=3000, p=2400, n=300)
        for i, seed in enumerate((1, 1, 2, 3)):
            ob = orc.fixed_rank_basis(g1, cfg.k, cfg.q, seed)
            h = r[f"h1_{i}"]
            e_ref = orc.sum_sq(ob.b)
            assert abs(h[0] ** 2 - h[1] ** 2 - e_ref) <= 1e-12 * e_ref, (i, seed)
            o = orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=seed)
            assert np.array_equal(r[f"alphas_{i}"], o.alphas)
            _, theta, _, _, _, _ = orc.comparative(o.alphas, o.betas, o.r)
            assert np.max(np.abs(r[f"theta_{i}"] - theta)) <= 1e-15


@pytest.mark.gpu
def test_sharded_single_process_matches_fused():
    import paper_2404_09459_b200 as rg

    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg)
    res = rdist.compute_gsv_sharded(torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda(),
                                    g1.shape[0], g2.shape[0], g1.shape[1], cfg.k, cfg.q, seed=0)
    run = rg.engine.run_device_pipeline(
        rg.GmpPair(g1, g2), rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q)))
    assert np.array_equal(res.alphas, run.alphas) and (res.r, res.s) == (run.r, run.s)
    assert res.residual_history1 == run.basis1.residual_history  # same kernels, same order
    assert res.residual_history2 == run.basis2.residual_history
