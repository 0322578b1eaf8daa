"""Row-sharded multi-GPU rGSVD.

G1 and G2 are split over ranks by contiguous row blocks (genes); every rank
holds ``g1[r0:r1]``, ``g2[s0:s1]`` in its own HBM. One process per GPU.
Each matrix chain is ONE native call per rank,
``rgsv_sketch_project_sharded`` (include/rgsv_b200.h), which runs the same
kernels as the single-GPU chain on the local rows and sums every cross-rank
partial in-stream through an all-reduce hook:

* Ω: generated on every rank from the same seed (identical, no traffic).
* ``||G||_F^2`` partial (1 value) -> all-reduce.
* shifted CholeskyQR3 of the row-sharded Y: each pass's k x k Gram partial
  -> all-reduce -> Cholesky + inverse redundantly on every rank (shift from
  the GLOBAL row count) -> local TRSM; Q stays row-sharded.
* power step: Zᵀ partial = Q_localᵀ G_local (kp x n) -> all-reduce; the wide
  CholeskyQR3 of the replicated Z runs redundantly; Y_local = G_local Q̂.
* projection: B partial -> all-reduce (B replicated, so ``||B||^2`` too).

The two chains run concurrently on two streams (G1 on the caller's stream,
G2 on a side stream), each with its own NCCL communicator so the two
streams never share one. After the join, rank 0 runs the small GSVD + the
comparative kernel and broadcasts the packed result (north_star: "the small
GSVD runs on one GPU and is broadcast"); every rank returns it.

Collectives (``Comm``):

* ``nccl``: communicators created inside librgsv_b200 (the 128-byte NCCL id
  is broadcast through torch.distributed), all-reduce = the library's
  ``rgsv_nccl_allreduce`` passed as the hook. Nothing touches the host
  between stages, so the whole sharded pair is captured as one CUDA graph
  (after one eager warm-up run) and replayed with new seeds.
* ``torch``: the hook is a host callback into ``torch.distributed`` (CPU
  staging). This is how the same native chain runs over gloo (the
  multi-process tests, several ranks on one GPU, where NCCL refuses
  duplicate devices).
* ``single``: one rank, no hook.

Traffic per power iteration for cfg2 (k = 120, n = 4000): 3 Gram
all-reduces of 131 KB and one 3.9 MB Zᵀ all-reduce, tiny next to the
per-rank GEMMs.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import device as _dev
from ._native import check, lib
from .errors import DimensionError, ValidationError

ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                ctypes.c_void_p)


def shard_rows(m: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row block [r0, r1) of an m-row matrix for `rank`."""
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


class _CudaView:
    """__cuda_array_interface__ over a raw device pointer (fp64 vector)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3, "strides": None}


class Comm:
    """The cross-rank sums and the broadcast of the sharded pipeline."""

    def __init__(self, mode: str = "auto", group=None):
        self.group = group
        init = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if init else 1
        self.rank = dist.get_rank(group) if init else 0
        if mode == "auto":
            if self.world == 1:
                mode = "single"
            elif dist.get_backend(group) == "nccl" and lib().rgsv_nccl_version() > 0:
                mode = "nccl"
            else:
                mode = "torch"
        if mode not in ("single", "nccl", "torch"):
            raise ValidationError(f"unknown comm mode {mode!r}")
        if mode != "single" and self.world == 1 and not init:
            raise ValidationError(f"comm mode {mode!r} needs an initialized process group")
        self.mode = mode
        self.comms = [None, None]
        self._cb = None
        if mode == "nccl":
            self._init_nccl()
        elif mode == "torch":
            self._cb = ALLREDUCE_FN(self._host_allreduce)

    # -- setup
    def _init_nccl(self):
        L = lib()
        ids = torch.zeros(256, dtype=torch.uint8)
        if self.rank == 0:
            for i in range(2):
                check(L.rgsv_nccl_get_unique_id(ctypes.c_void_p(ids.data_ptr() + 128 * i)),
                      "rgsv_nccl_get_unique_id")
        dev_ids = ids.cuda() if dist.get_backend(self.group) == "nccl" else ids
        dist.broadcast(dev_ids, 0, group=self.group)
        ids = dev_ids.cpu()
        for i in range(2):  # one communicator per chain stream
            c = ctypes.c_void_p()
            check(L.rgsv_nccl_comm_init(ctypes.byref(c), self.world,
                                        ctypes.c_void_p(ids.data_ptr() + 128 * i), self.rank),
                  "rgsv_nccl_comm_init")
            self.comms[i] = c

    def close(self):
        for i, c in enumerate(self.comms):
            if c is not None:
                lib().rgsv_nccl_comm_destroy(c)
                self.comms[i] = None

    # -- the hook handed to rgsv_sketch_project_sharded
    def hook(self, chain: int):
        """(fn, ctx) for chain 0 (G1) or 1 (G2)."""
        if self.mode == "single":
            return ctypes.c_void_p(0), ctypes.c_void_p(0)
        if self.mode == "nccl":
            return ctypes.cast(lib().rgsv_nccl_allreduce, ctypes.c_void_p), self.comms[chain]
        return ctypes.cast(self._cb, ctypes.c_void_p), ctypes.c_void_p(0)

    def _host_allreduce(self, buf, count, stream, ctx) -> int:
        try:
            st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
            st.synchronize()
            t = torch.as_tensor(_CudaView(buf, int(count)), device="cuda")
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            with torch.cuda.stream(st):
                t.copy_(h)
            st.synchronize()
            return 0
        except Exception:  # surfaced as RGSV_ERR_CUDA by the caller
            return 1

    # -- tensor-level collectives (the fp32 chain, the packed broadcast)
    def allreduce_tensor(self, t: torch.Tensor, chain: int = 0) -> torch.Tensor:
        if self.mode == "single":
            return t
        if self.mode == "nccl":
            check(lib().rgsv_nccl_allreduce(_dev.vp(t), t.numel(),
                                            _dev.sp(torch.cuda.current_stream()),
                                            self.comms[chain]), "rgsv_nccl_allreduce")
            return t
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
        if h is not t:
            t.copy_(h)
        return t

    def broadcast(self, t: torch.Tensor, root: int = 0) -> None:
        if self.mode == "single":
            return
        if self.mode == "nccl":
            check(lib().rgsv_nccl_broadcast(_dev.vp(t), t.numel() * t.element_size(), root,
                                            _dev.sp(torch.cuda.current_stream()),
                                            self.comms[0]), "rgsv_nccl_broadcast")
            return
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        h = t.cpu()
        dist.broadcast(h, root, group=self.group)
        if h is not t:
            t.copy_(h)


class ShardedPairPlan:
    """Buffers, streams and (NCCL mode) the captured CUDA graph for one
    row-sharded fp64 pair shape on this rank."""

    def __init__(self, comm: Comm, m_local: int, p_local: int, m: int, p: int, n: int,
                 k1: int, k2: int):
        self.comm = comm
        self.m_local, self.p_local, self.m, self.p, self.n = m_local, p_local, m, p, n
        self.k1, self.k2 = k1, k2
        self.s1 = _dev.SketchPlan(m_local, n, k1)
        self.s2 = _dev.SketchPlan(p_local, n, k2)
        self.small_bytes = int(lib().rgsv_small_gsvd_workspace_bytes(k1, k2, n))
        self.small_ws = torch.empty(self.small_bytes, dtype=torch.uint8, device="cuda")
        self.pk = _dev._Packed(n, k1, k2)
        self.side = torch.cuda.Stream()
        self.graph = None
        self.graph_key = None
        self.last_key = None
        self.kernels_per_replay = 0

    def _chain(self, sub, g, rows_total: int, q_iters: int, stats, rdiag, status, chain, stream):
        fn, ctx = self.comm.hook(chain)
        rc = lib().rgsv_sketch_project_sharded(
            _dev.vp(g.t), g.ld, g.rows, rows_total, g.cols, _dev.vp(sub.om_dev), sub.ldb, sub.k,
            q_iters, _dev.vp(sub.q), _dev.vp(sub.b), sub.ldb, _dev.vp(stats), _dev.vp(rdiag),
            _dev.vp(status), fn, ctx, _dev.vp(sub.ws), sub.ws_bytes, _dev.sp(stream))
        check(rc, "rgsv_sketch_project_sharded")

    def enqueue(self, g1, g2, q_iters: int, classify_tol: float) -> None:
        L = lib()
        main = torch.cuda.current_stream()
        pk = self.pk
        pk.d("status").zero_()
        self.side.wait_stream(main)
        self.s1.enqueue_omega(pk.d("status"), main)
        self.s2.enqueue_omega(pk.d("status"), self.side)
        self._chain(self.s1, g1, self.m, q_iters, pk.d("stats1"), pk.d("rdiag1"), pk.d("status"),
                    0, main)
        with torch.cuda.stream(self.side):
            self._chain(self.s2, g2, self.p, q_iters, pk.d("stats2"), pk.d("rdiag2"),
                        pk.d("status"), 1, self.side)
        main.wait_stream(self.side)
        if self.comm.rank == 0:
            rc = L.rgsv_small_gsvd(_dev.vp(self.s1.b), self.s1.ldb, self.k1, _dev.vp(self.s2.b),
                                   self.s2.ldb, self.k2, self.n, _dev.vp(pk.d("sv1")),
                                   _dev.vp(pk.d("sv2")), _dev.vp(pk.d("nsv")),
                                   _dev.vp(pk.d("status")), _dev.vp(self.small_ws),
                                   self.small_bytes, _dev.sp(main))
            check(rc, "rgsv_small_gsvd")
            rc = L.rgsv_comparative(_dev.vp(pk.d("sv1")), _dev.vp(pk.d("nsv")),
                                    _dev.vp(pk.d("sv2")), self.n, float(classify_tol),
                                    _dev.vp(pk.d("alphas")), _dev.vp(pk.d("betas")),
                                    _dev.vp(pk.d("rho")), _dev.vp(pk.d("theta")),
                                    _dev.vp(pk.d("p1")), _dev.vp(pk.d("p2")),
                                    _dev.vp(pk.d("scalars")), _dev.vp(pk.d("counts")),
                                    _dev.vp(pk.d("status")), _dev.sp(main))
            check(rc, "rgsv_comparative")
        self.comm.broadcast(pk.dev, 0)  # the small GSVD's result to every rank
        pk.host.copy_(pk.dev, non_blocking=True)

    def run(self, g1, g2, seed: int, q_iters: int, classify_tol: float, sync: bool = True):
        """Seeds of the reference convention (seed for G1, seed + 1 for G2,
        engine.py:252-253). NCCL mode: eager on the first sighting of a
        buffer set, captured on the second, replayed after (the bench's
        timed path); the torch (host-callback) mode is always eager."""
        self.s1.set_seed(seed)
        self.s2.set_seed(int(seed) + 1)
        key = (g1.t.data_ptr(), g1.ld, g1.rows, g2.t.data_ptr(), g2.ld, g2.rows, int(q_iters),
               float(classify_tol))
        graphs = _dev.USE_GRAPHS and self.comm.mode in ("nccl", "single")
        if self.graph is not None and self.graph_key == key:
            self.graph.replay()
            _dev.GRAPH_REPLAYS[0] += 1
            _dev.GRAPH_REPLAYS[1] += self.kernels_per_replay
        elif graphs and self.last_key == key:
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            n0 = lib().rgsv_launch_count()
            with torch.cuda.graph(graph):
                self.enqueue(g1, g2, q_iters, classify_tol)
            self.kernels_per_replay = lib().rgsv_launch_count() - n0
            self.graph, self.graph_key = graph, key
            graph.replay()
            _dev.GRAPH_REPLAYS[0] += 1
            _dev.GRAPH_REPLAYS[1] += self.kernels_per_replay
        else:
            self.enqueue(g1, g2, q_iters, classify_tol)
        self.last_key = key
        if sync:
            torch.cuda.current_stream().synchronize()
        return self.pk


@dataclass
class ShardedResult:
    alphas: np.ndarray
    betas: np.ndarray
    r: int
    s: int
    residual_history1: list
    residual_history2: list
    b1: object  # replicated projections (device, kp x ldn)
    b2: object
    report: object = None  # the engine.DeviceRun (rho, theta, P, D, status)


_PLANS: dict = {}
_COMMS: dict = {}


def default_comm(mode: str = "auto") -> Comm:
    """One Comm per (process group, mode), created collectively on first use."""
    init = dist.is_available() and dist.is_initialized()
    key = (id(dist.group.WORLD) if init else None, mode)
    c = _COMMS.get(key)
    if c is None:
        c = Comm(mode)
        _COMMS[key] = c
    return c


def sharded_plan(comm: Comm, m_local, p_local, m, p, n, k1, k2) -> ShardedPairPlan:
    key = (id(comm), torch.cuda.current_device(), m_local, p_local, m, p, n, k1, k2)
    plan = _PLANS.get(key)
    if plan is None:
        if len(_PLANS) > 4:
            _PLANS.clear()
        plan = ShardedPairPlan(comm, m_local, p_local, m, p, n, k1, k2)
        _PLANS[key] = plan
    return plan


def _f32_chain(comm: Comm, g, rows_total: int, k: int, q: int, seed: int, chain: int):
    """One fp32 row shard through the tf32x3 tensor-core chain
    (tf32.tf32_chain) with every partial summed over the ranks."""
    from . import tf32 as _tf32

    lo = torch.empty((g.rows, g.ld), dtype=torch.float32, device="cuda")
    _, b, hist = _tf32.tf32_chain(g, k, q, seed, lo=lo,
                                  reduce=lambda t: comm.allreduce_tensor(t, chain),
                                  rows_total=rows_total)
    del lo
    return b, hist


def compute_gsv_sharded(g1_local, g2_local, m: int, p: int, n: int, k: int, q: int = 0,
                        seed: int = 0, classify_tol: float = 1e-10, comm: Comm | None = None,
                        sync: bool = True) -> ShardedResult:
    """Row-sharded compute_gsv + compare for the fixed-rank pipeline.
    `g1_local` / `g2_local` are this rank's row blocks (see shard_rows) as
    CUDA tensors. Every rank returns the same result (broadcast from rank 0).
    fp64 shards run the native sharded chain; an fp32 shard runs the
    tf32x3 tensor-core chain (chosen per matrix, by its own dtype)."""
    from .engine import GsvOptions, unpack
    from .rangefinder import ExtractionConfig

    comm = comm or default_comm()
    a = _dev.to_device(g1_local, "g1_local", keep_f32=True)
    b = _dev.to_device(g2_local, "g2_local", keep_f32=True)
    if a.cols != n or b.cols != n:
        raise DimensionError(f"shards must have n={n} columns, got {a.cols} and {b.cols}")
    if k > min(m, n) or k > min(p, n):
        raise ValidationError(f"max_cols={k} exceeds min(rows, cols)")
    if m + p < n:
        raise ValidationError(f"stacked pair has {m + p} rows < {n} columns")
    opts = GsvOptions(extraction=ExtractionConfig.fixed_rank(k, seed, q),
                      classify_tol=classify_tol)
    if not a.is_f32 and not b.is_f32 and _dev.ceil16(k) <= 128:
        plan = sharded_plan(comm, a.rows, b.rows, m, p, n, k, k)
        pk = plan.run(a, b, seed, q, classify_tol, sync=True)
        run = unpack(pk, plan, opts)  # status bits -> reference exceptions, GsvSpectrum
        return ShardedResult(run.alphas, run.betas, run.r, run.s,
                             run.basis1.residual_history, run.basis2.residual_history,
                             plan.s1.b, plan.s2.b, run)
    # per-matrix chains: fp32 shards on the tf32x3 tensor cores, fp64 (wide
    # k) through the native sharded chain as a one-off plan
    outs = []
    for chain, (g, rows_total, sd) in enumerate(((a, m, seed), (b, p, seed + 1))):
        if g.is_f32:
            outs.append(_f32_chain(comm, g, rows_total, k, q, sd, chain))
        else:
            sub = _dev.SketchPlan(g.rows, n, k)
            sub.set_seed(sd)
            stats = torch.zeros(2, dtype=torch.float64, device="cuda")
            rdiag = torch.zeros(max(k, 1), dtype=torch.float64, device="cuda")
            status = torch.zeros(1, dtype=torch.int32, device="cuda")
            st = torch.cuda.current_stream()
            sub.enqueue_omega(status, st)
            fn, ctx = comm.hook(chain)
            check(lib().rgsv_sketch_project_sharded(
                _dev.vp(g.t), g.ld, g.rows, rows_total, n, _dev.vp(sub.om_dev), sub.ldb, k, q,
                _dev.vp(sub.q), _dev.vp(sub.b), sub.ldb, _dev.vp(stats), _dev.vp(rdiag),
                _dev.vp(status), fn, ctx, _dev.vp(sub.ws), sub.ws_bytes, _dev.sp(st)),
                "rgsv_sketch_project_sharded")
            gf2, e = (float(x) for x in stats.cpu())
            outs.append((sub.b, [math.sqrt(gf2), math.sqrt(max(gf2 - e, 0.0))]))
    (b1, h1), (b2, h2) = outs
    for h in (h1, h2):
        if not math.isfinite(h[0]):
            raise ValidationError("g contains non-finite entries")
    from .engine import _small_checked

    out = _small_checked(b1, k, b2, k, n, classify_tol)
    r, s = out["counts"]
    from .engine import GsvSpectrum

    spec = GsvSpectrum(out["alphas"], out["betas"], r, s)
    return ShardedResult(spec.alphas, spec.betas, r, s, h1, h2, b1, b2, out)


__all__ = ["shard_rows", "Comm", "ShardedPairPlan", "compute_gsv_sharded", "ShardedResult",
           "default_comm", "sharded_plan"]
