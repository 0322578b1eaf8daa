"""Row-sharded multi-rank driver (paper_2404_09459_b200/dist.py).

CPU: world_size 2 over gloo with a torch-CPU stand-in for the local kernels
(test-only), checked against the oracle: the sharding and the collective
sequence must reproduce the single-process result. GPU: the same driver on
the CUDA backend at world_size 1 against the fused pipeline.
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


class TorchCpuBackend:
    """Reference stand-in for the device kernels (float64 on the CPU)."""

    def zeros(self, *shape):
        return torch.zeros(shape, dtype=torch.float64)

    def to_host(self, t):
        return t.numpy()

    def omega_t(self, n, k, seed, kp, ldn):
        om = torch.zeros((kp, ldn), dtype=torch.float64)
        om[:k, :n] = torch.from_numpy(orc.gaussian_matrix(n, k, seed).T.copy())
        return om

    def gx(self, a, bt, M, N, K, out, max_split=32):
        out[:M, :N] = a[:M, :K] @ bt[:N, :K].T

    def gtq(self, a, b, M, N, K, out):
        out[:M, :N] = a[:K, :M].T @ b[:K, :N]

    def chol_inv(self, gram, k, kp, shift_rows):
        a = gram[:k, :k].clone()
        if shift_rows > 0:
            tr = float(torch.trace(a))
            a += 11.0 * (shift_rows * k + k * (k + 1)) * 2.0 ** -53 * tr * torch.eye(k, dtype=a.dtype)
        lo = torch.linalg.cholesky(a)
        li = torch.linalg.inv(lo)
        linv = torch.eye(kp, dtype=torch.float64)
        linv[:k, :k] = li
        return linv, linv.T.contiguous()

    def sumsq(self, a, rows, cols):
        return torch.tensor([float((a[:rows, :cols] ** 2).sum())], dtype=torch.float64)

    def spectrum(self, b1, b2, k1, k2, n, classify_tol):
        s = np.vstack([b1[:k1, :n].numpy(), b2[:k2, :n].numpy()])
        qf, _ = orc.reduced_qr(s)
        al, be, r, s_, _, _ = orc.spectrum_from_l_blocks(qf[:k1], qf[k1:], n, classify_tol)
        return al, be, r, s_, 0


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg, m=700, p=500)
    m, p, n = g1.shape[0], g2.shape[0], g1.shape[1]
    r0, r1 = rdist.shard_rows(m, rank, world)
    s0, s1 = rdist.shard_rows(p, rank, world)
    res = rdist.compute_gsv_sharded(torch.from_numpy(g1[r0:r1].copy()),
                                    torch.from_numpy(g2[s0:s1].copy()), m, p, n, cfg.k, cfg.q,
                                    seed=3, backend=TorchCpuBackend())
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), alphas=res.alphas, betas=res.betas,
             rs=np.array([res.r, res.s]), h1=np.array(res.residual_history1),
             h2=np.array(res.residual_history2), b1=res.b1.numpy())
    dist.destroy_process_group()


def test_shard_rows_cover():
    for m in (1, 7, 20000, 200000):
        for w in (1, 2, 3, 8):
            blocks = [rdist.shard_rows(m, r, w) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in blocks) - min(b - a for a, b in blocks) <= 1


def test_two_rank_gloo_matches_oracle():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        r0 = np.load(os.path.join(d, "r0.npz"))
        r1 = np.load(os.path.join(d, "r1.npz"))
        for key in ("alphas", "betas", "rs", "h1", "h2", "b1"):
            assert np.array_equal(r0[key], r1[key]), key  # replicated results agree
        cfg = CONFIGS["cfg0"]
        g1, g2 = make_pair(cfg, m=700, p=500)
        o = orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=3)
        assert np.array_equal(r0["alphas"], o.alphas) and list(r0["rs"]) == [o.r, o.s]
        h = r0["h1"]
        e_ref = orc.sum_sq(o.basis1.b)
        assert abs(h[0] - o.basis1.residual_history[0]) <= 1e-13 * h[0]
        assert abs(h[0] ** 2 - h[1] ** 2 - e_ref) <= 1e-12 * e_ref
        # leading signal rows of B agree with the oracle's (same phase convention)
        b_ref = o.basis1.b
        s = cfg.s
        assert np.linalg.norm(r0["b1"][:s, : g1.shape[1]] - b_ref[:s]) <= 1e-11 * np.linalg.norm(b_ref[:s])


@pytest.mark.gpu
def test_sharded_driver_on_device_matches_fused():
    import paper_2404_09459_b200 as rg

    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg)
    res = rdist.compute_gsv_sharded(torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda(),
                                    g1.shape[0], g2.shape[0], g1.shape[1], cfg.k, cfg.q, seed=0)
    run = rg.engine.run_device_pipeline(
        rg.GmpPair(g1, g2), rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q)))
    assert np.array_equal(res.alphas, run.alphas) and (res.r, res.s) == (run.r, run.s)
    e_s = res.residual_history1[0] ** 2 - res.residual_history1[1] ** 2
    e_f = run.basis1.residual_history[0] ** 2 - run.basis1.residual_history[1] ** 2
    assert abs(e_s - e_f) <= 1e-12 * e_f
    assert math.isclose(res.residual_history1[0], run.basis1.residual_history[0], rel_tol=1e-14)
