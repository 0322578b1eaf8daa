"""Row-sharded multi-GPU rGSVD.

G1 and G2 are split over ranks by contiguous row blocks (genes); every rank
holds `g1[r0:r1]`, `g2[s0:s1]` in its own HBM. One process per GPU,
``torch.distributed`` over NCCL. Per matrix chain:

* Ω: generated on every rank from the same seed (identical, no traffic).
* Y_local = G_local Ω (local DMMA GEMM); ||G||_F^2 partial -> all-reduce.
* shifted CholeskyQR3 on the row-sharded Y: per pass the k x k Gram partial
  Y_localᵀ Y_local -> all-reduce -> Cholesky + inverse redundantly on every
  rank -> local TRSM (Q stays row-sharded).
* power step: Zᵀ partial = Q_localᵀ G_local (k x n) -> all-reduce; the wide
  QR of the replicated Z runs redundantly; Y_local = G_local Q̂.
* projection: B partial = Q_localᵀ G_local -> all-reduce (B replicated).
* the small GSVD and the comparative kernel run redundantly on every rank,
  so every rank returns the same spectrum (no broadcast needed).

Traffic per power iteration for cfg2 (k = 120, n = 4000): 3 Gram
all-reduces of 131 KB and one 3.9 MB Zᵀ all-reduce — latency-bound, tiny
next to the per-rank GEMMs. The local operations go through a backend
object: ``CudaBackend`` (the C-ABI kernels, the product) or any object with
the same methods (the CPU tests inject a numpy one to check the sharding and
collective choreography on gloo).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import device as _dev
from ._native import ST_CHOL, ST_JACOBI, ST_OMEGA_SHORT, check, lib
from .errors import ConvergenceError, RankDeficiencyError, ValidationError


def shard_rows(m: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row block [r0, r1) of an m-row matrix for `rank`."""
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


class CudaBackend:
    """Local operations of the sharded pipeline on the B200 kernels."""

    def __init__(self):
        _dev.require_device()
        self.L = lib()
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    # -- helpers
    def _st(self):
        return _dev.sp(torch.cuda.current_stream())

    def zeros(self, *shape):
        return torch.zeros(shape, dtype=torch.float64, device="cuda")

    def to_host(self, t):
        return t.cpu().numpy()

    def omega_t(self, n: int, k: int, seed: int, kp: int, ldn: int):
        return _dev.omega_device(n, k, [seed], ldo=ldn)[0]

    def gx(self, a, bt, M: int, N: int, K: int, out, max_split: int = 32):
        """out (M x N) = a (M x K) bt^T."""
        check(self.L.rgsv_gemm_gx(_dev.vp(a), a.stride(0), _dev.vp(bt), bt.stride(0),
                                  _dev.vp(out), out.stride(0), M, N, K, _dev.vp(self.scratch),
                                  self.scratch.numel(), self._st()), "gemm_gx")

    def gtq(self, a, b, M: int, N: int, K: int, out):
        """out (M x N) = a^T b, a: K x M, b: K x N."""
        check(self.L.rgsv_gemm_gtq(_dev.vp(a), a.stride(0), _dev.vp(b), b.stride(0),
                                   _dev.vp(out), out.stride(0), M, N, K, _dev.vp(self.scratch),
                                   self.scratch.numel(), self._st()), "gemm_gtq")

    def chol_inv(self, gram, k: int, kp: int, shift_rows: int):
        linv = torch.zeros(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
        rinv = self.zeros(kp, kp)
        rdiag = self.zeros(kp)
        check(self.L.rgsv_chol_inv(_dev.vp(gram), k, kp, shift_rows, _dev.vp(linv),
                                   _dev.vp(rinv), _dev.vp(rdiag), _dev.vp(self.status),
                                   self._st()), "chol_inv")
        return linv[: kp * kp].view(kp, kp), rinv

    def sumsq(self, a, rows: int, cols: int) -> torch.Tensor:
        out = self.zeros(1)
        ws = self.zeros(1024)
        check(self.L.rgsv_sumsq(_dev.vp(a), a.stride(0), rows, cols, _dev.vp(out), _dev.vp(ws),
                                ws.numel() * 8, self._st()), "sumsq")
        return out

    def spectrum(self, b1, b2, k1: int, k2: int, n: int, classify_tol: float):
        """Small GSVD + comparative kernel; returns host arrays."""
        L = self.L
        nb = int(L.rgsv_small_gsvd_workspace_bytes(k1, k2, n))
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        sv1 = self.zeros(max(k1, 1))
        sv2 = self.zeros(max(k2, 1))
        ints = torch.zeros(8, dtype=torch.int32, device="cuda")
        check(L.rgsv_small_gsvd(_dev.vp(b1), b1.stride(0), k1, _dev.vp(b2), b2.stride(0), k2, n,
                                _dev.vp(sv1), _dev.vp(sv2), _dev.vp(ints[0:2]),
                                _dev.vp(self.status), _dev.vp(ws), nb, self._st()), "small_gsvd")
        res = self.zeros(6 * n + 4)
        check(L.rgsv_comparative(_dev.vp(sv1), _dev.vp(ints[0:2]), _dev.vp(sv2), n,
                                 float(classify_tol), *(_dev.vp(res[i * n:(i + 1) * n])
                                                        for i in range(6)),
                                 _dev.vp(res[6 * n:]), _dev.vp(ints[2:4]), _dev.vp(self.status),
                                 self._st()), "comparative")
        h = res.cpu().numpy()
        iv = ints.cpu().numpy()
        code = int(self.status.item())
        return h[:n].copy(), h[n:2 * n].copy(), int(iv[2]), int(iv[3]), code


@dataclass
class ShardedResult:
    alphas: np.ndarray
    betas: np.ndarray
    r: int
    s: int
    residual_history1: list
    residual_history2: list
    b1: object  # replicated projections (backend arrays)
    b2: object


def _all_reduce(t):
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def sharded_cholqr3(be, y, rows_total: int, m_local: int, k: int, kp: int):
    """Shifted CholeskyQR3 of a row-sharded tall Y (m_local x kp per rank)."""
    for step in range(3):
        gram = be.zeros(kp, kp)
        if m_local > 0:
            be.gtq(y, y, kp, kp, m_local, gram)
        _all_reduce(gram)
        linv, _ = be.chol_inv(gram, k, kp, rows_total if step == 0 else 0)
        q = be.zeros(max(m_local, 1), kp)
        if m_local > 0:
            be.gx(y, linv, m_local, kp, kp, q, max_split=1)
        y = q
    return y


def wide_cholqr3(be, bt, n: int, ldn: int, k: int, kp: int):
    """Shifted CholeskyQR3 of Z = B^T given B (kp x n), replicated: returns
    Qhat^T (kp x ldn)."""
    src = bt
    for step in range(3):
        gram = be.zeros(kp, kp)
        be.gx(src, src, kp, kp, n, gram)
        _, rinv = be.chol_inv(gram, k, kp, n if step == 0 else 0)
        dst = be.zeros(kp, ldn)
        be.gtq(rinv, src, kp, n, kp, dst)
        src = dst
    return src


def sharded_chain(be, g_local, m_total: int, m_local: int, n: int, k: int, q: int, seed: int):
    """One matrix chain on the row-sharded G (g_local: m_local x n)."""
    kp = _dev.ceil16(k)
    ldn = _dev.ceil16(n)
    om = be.omega_t(n, k, seed, kp, ldn)
    ss = be.sumsq(g_local, m_local, n) if m_local > 0 else be.zeros(1)
    _all_reduce(ss)
    y = be.zeros(max(m_local, 1), kp)
    if m_local > 0:
        be.gx(g_local, om, m_local, kp, n, y)
    qb = sharded_cholqr3(be, y, m_total, m_local, k, kp)
    for _ in range(q):
        zt = be.zeros(kp, ldn)
        if m_local > 0:
            be.gtq(qb, g_local, kp, n, m_local, zt)
        _all_reduce(zt)
        qht = wide_cholqr3(be, zt, n, ldn, k, kp)
        y = be.zeros(max(m_local, 1), kp)
        if m_local > 0:
            be.gx(g_local, qht, m_local, kp, n, y)
        qb = sharded_cholqr3(be, y, m_total, m_local, k, kp)
    b = be.zeros(kp, ldn)
    if m_local > 0:
        be.gtq(qb, g_local, kp, n, m_local, b)
    _all_reduce(b)
    gf2 = float(be.to_host(ss)[0])
    energy = float(be.to_host(be.sumsq(b, kp, n))[0])
    return b, gf2, energy


def sharded_chain_f32(be, g_local, m_total: int, n: int, k: int, q: int, seed: int, lo=None):
    """One matrix chain on a row-sharded fp32 G: the tf32x3 tensor-core chain
    (tf32.tf32_chain) with every k x k Gram, Z^T, B and ||G||^2 partial
    all-reduced over the ranks."""
    from . import tf32 as _tf32

    a = _dev.to_device(g_local, "g_local", keep_f32=True)
    _, b, hist = _tf32.tf32_chain(a, k, q, seed, lo=lo, reduce=_all_reduce, rows_total=m_total)
    energy = float(be.sumsq(b, b.shape[0], n).cpu()[0])
    return b, hist[0] ** 2, energy


def _is_f32_cuda(t) -> bool:
    return isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32


def compute_gsv_sharded(g1_local, g2_local, m: int, p: int, n: int, k: int, q: int = 0,
                        seed: int = 0, classify_tol: float = 1e-10, backend=None):
    """Row-sharded compute_gsv for the fixed-rank pipeline. `g1_local` /
    `g2_local` are this rank's row blocks (see shard_rows). Every rank
    returns the same ShardedResult. fp32 CUDA shards (cfg4) take the
    tensor-core tf32x3 chain; fp64 shards the DMMA chain."""
    be = backend or CudaBackend()
    if k > min(m, n) or k > min(p, n):
        raise ValidationError(f"max_cols={k} exceeds min(rows, cols)")
    m_local = g1_local.shape[0]
    p_local = g2_local.shape[0]
    if backend is None and _is_f32_cuda(g1_local) and _is_f32_cuda(g2_local):
        lo = torch.empty(max(g1_local.numel(), g2_local.numel()), dtype=torch.float32,
                         device="cuda")
        b1, gf1, e1 = sharded_chain_f32(be, g1_local, m, n, k, q, seed,
                                        lo=lo[: g1_local.numel()].view(g1_local.shape))
        b2, gf2, e2 = sharded_chain_f32(be, g2_local, p, n, k, q, seed + 1,
                                        lo=lo[: g2_local.numel()].view(g2_local.shape))
        del lo
    else:
        b1, gf1, e1 = sharded_chain(be, g1_local, m, m_local, n, k, q, seed)
        b2, gf2, e2 = sharded_chain(be, g2_local, p, p_local, n, k, q, seed + 1)
    alphas, betas, r, s, code = be.spectrum(b1, b2, k, k, n, classify_tol)
    if code & ST_OMEGA_SHORT:
        raise RuntimeError("device Omega generator exhausted its draw margin")
    if code & ST_CHOL:
        raise RankDeficiencyError("CholeskyQR breakdown in the sharded pipeline")
    if code & ST_JACOBI:
        raise ConvergenceError("Jacobi SVD did not converge")
    h1 = [math.sqrt(gf1), math.sqrt(max(gf1 - e1, 0.0))]
    h2 = [math.sqrt(gf2), math.sqrt(max(gf2 - e2, 0.0))]
    return ShardedResult(alphas, betas, r, s, h1, h2, b1, b2)


__all__ = ["shard_rows", "CudaBackend", "compute_gsv_sharded", "ShardedResult",
           "sharded_cholqr3", "wide_cholqr3", "sharded_chain", "sharded_chain_f32"]
