"""Device-side orchestration of the rGSVD hot path.

Owns the device buffers of a pair (cached per shape in a ``PairPlan``),
issues the C-ABI calls on CUDA streams, and brings every small result back
in ONE device->host copy. Matrices live in HBM as row-major float64 with an
even row pitch (TMA needs 16-byte pitches); bases are padded to
kp = ceil16(k) columns with exact zeros.

Stream layout for a pair: the G1 chain (sketch -> CholQR3 -> q power
iterations -> projection) runs on the caller's stream and the G2 chain on
a side stream concurrently, so the single-CTA Cholesky steps of one chain
overlap the DMMA GEMMs of the other; the small GSVD and the fused
comparative kernel run after the join.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._native import check, lib, require_device
from .errors import DimensionError, ValidationError

SEED_MASK = (1 << 64) - 1
F64 = torch.float64


def ceil16(x: int) -> int:
    return (x + 15) // 16 * 16


def vp(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def sp(stream: torch.cuda.Stream) -> ctypes.c_void_p:
    return ctypes.c_void_p(stream.cuda_stream)


@dataclass
class DevMatrix:
    """Row-major float64 matrix in HBM: ``t`` is a rows x cols view whose row
    stride ``ld`` is even (TMA row pitch)."""

    t: torch.Tensor
    rows: int
    cols: int

    @property
    def ld(self) -> int:
        return self.t.stride(0)

    @property
    def is_f32(self) -> bool:
        return self.t.dtype == torch.float32


def _even(x: int) -> int:
    return x + (x & 1)


def to_device(a, name: str = "matrix", keep_f32: bool = False) -> DevMatrix:
    """Validate shape/field like core.as_matrix (core.py:43-57) and place
    the matrix in HBM (no copy when it already is a suitable CUDA tensor).
    Finiteness is checked on the device by the fused sum-of-squares pass.
    keep_f32: float32 input stays float32 in HBM (the cfg4 path promotes it
    to fp64 chunk by chunk, exactly like the reference's up-front
    promotion, core.py:51-54, but without a second full-size copy)."""
    require_device()
    if isinstance(a, DevMatrix):
        return a
    is32 = (isinstance(a, torch.Tensor) and a.dtype == torch.float32) or \
        (not isinstance(a, torch.Tensor) and np.asarray(a).dtype == np.float32)
    if keep_f32 and is32:
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        if t.dim() != 2 or t.shape[0] < 1 or t.shape[1] < 1:
            raise DimensionError(f"{name} must be 2-D with positive dimensions, got "
                                 f"{tuple(t.shape)}")
        if t.device.type != "cuda" or t.stride(1) != 1:
            t = t.to("cuda").contiguous()
        return DevMatrix(t, t.shape[0], t.shape[1])
    if isinstance(a, torch.Tensor):
        t = a
        if t.dim() != 2:
            raise DimensionError(f"{name} must be 2-D, got shape {tuple(t.shape)}")
        rows, cols = t.shape
        if rows < 1 or cols < 1:
            raise DimensionError(f"{name} must have positive dimensions, got {tuple(t.shape)}")
        if t.is_complex():
            raise ValidationError(f"{name}: complex matrices are not supported by the B200 path")
        if t.dtype != F64:
            t = t.to(F64)
        if t.device.type != "cuda":
            t = t.to("cuda")
        if (t.stride(1) == 1 and t.stride(0) >= cols and t.stride(0) % 2 == 0
                and t.data_ptr() % 16 == 0):
            return DevMatrix(t, rows, cols)
        dev = torch.zeros((rows, _even(cols)), dtype=F64, device="cuda")
        dev[:, :cols].copy_(t)
        return DevMatrix(dev[:, :cols], rows, cols)
    arr = np.asarray(a)
    if arr.ndim != 2:
        raise DimensionError(f"{name} must be 2-D, got shape {arr.shape}")
    if arr.shape[0] < 1 or arr.shape[1] < 1:
        raise DimensionError(f"{name} must have positive dimensions, got {arr.shape}")
    if np.iscomplexobj(arr):
        raise ValidationError(f"{name}: complex matrices are not supported by the B200 path")
    rows, cols = arr.shape
    host = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
    if cols % 2 == 0:
        dev = torch.empty((rows, cols), dtype=F64, device="cuda")
        dev.copy_(host, non_blocking=host.is_pinned())
    else:
        dev = torch.zeros((rows, cols + 1), dtype=F64, device="cuda")
        dev[:, :cols].copy_(host)
        dev = dev[:, :cols]
    return DevMatrix(dev, rows, cols)


def seed_word(seed: int) -> int:
    """The reference's seed convention, seed & (2^64 - 1) (rangefinder.py:101),
    as the two's-complement int64 a torch tensor can hold."""
    v = int(seed) & SEED_MASK
    return v - (1 << 64) if v >= (1 << 63) else v


def omega_device(n: int, k: int, seeds, ldo: int | None = None) -> torch.Tensor:
    """Omega^T blocks (len(seeds) x kp x ldo) drawn on the device, bit-identical
    to default_rng(seed).standard_normal((n, k)) (rgsv_omega_generate)."""
    require_device()
    kp = ceil16(k)
    ldo = ldo or ceil16(n)
    seeds = list(seeds)
    ns = len(seeds)
    out = torch.zeros((ns, kp, ldo), dtype=F64, device="cuda")
    sd = torch.tensor([seed_word(x) for x in seeds], dtype=torch.int64).cuda()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    nb = int(lib().rgsv_omega_workspace_bytes(ns, n, k))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    check(lib().rgsv_omega_generate(vp(sd), ns, n, k, vp(out), ldo, kp * ldo, vp(status), vp(ws),
                                    nb, sp(torch.cuda.current_stream())), "rgsv_omega_generate")
    if int(status.item()) & _native.ST_OMEGA_SHORT:
        raise RuntimeError("Omega generator exhausted its draw margin")
    return out


def omega_block(n: int, width: int, seed: int, offset: int, ldo: int) -> torch.Tensor:
    """Omega^T (ceil16(width) x ldo) of block i of the adaptive range finder:
    the n x width normals drawn from default_rng(seed) after `offset` earlier
    normals (rangefinder.py:101,112), generated on the device."""
    kp = ceil16(width)
    out = torch.zeros((kp, ldo), dtype=F64, device="cuda")
    sd = torch.tensor([seed_word(seed)], dtype=torch.int64).cuda()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    nb = int(lib().rgsv_omega_workspace_bytes_at(1, n, width, offset))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    check(lib().rgsv_omega_generate_at(vp(sd), 1, n, width, offset, vp(out), ldo, kp * ldo,
                                       vp(status), vp(ws), nb, sp(torch.cuda.current_stream())),
          "rgsv_omega_generate_at")
    if int(status.item()) & _native.ST_OMEGA_SHORT:
        raise RuntimeError("Omega generator exhausted its draw margin")
    return out


def small_spectrum(b1: torch.Tensor, l1: int, b2: torch.Tensor, l2: int, n: int,
                   classify_tol: float) -> dict:
    """Stacked QR + L-block singular values + fused comparative kernel for
    arbitrary compressed blocks b1 (l1 x n), b2 (l2 x n) in HBM (row-major,
    even pitch) -- engine.py:257-261 + :189-225 + analysis.py:82-102.
    Returns host arrays (one D2H copy)."""
    L = lib()
    st = sp(torch.cuda.current_stream())
    nb = int(L.rgsv_small_gsvd_workspace_bytes(l1, l2, n))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    res = torch.zeros(6 * n + 4 + 2 * max(l1, l2, 1) + 4, dtype=F64, device="cuda")
    sv1 = res[6 * n + 4: 6 * n + 4 + max(l1, l2, 1)]
    sv2 = res[6 * n + 4 + max(l1, l2, 1): 6 * n + 4 + 2 * max(l1, l2, 1)]
    ints = torch.zeros(8, dtype=torch.int32, device="cuda")
    status = ints[4:5]
    dummy = torch.zeros(2, dtype=F64, device="cuda")
    pb1 = vp(b1) if l1 else vp(dummy)
    pb2 = vp(b2) if l2 else vp(dummy)
    ld1 = b1.stride(0) if l1 else 2
    ld2 = b2.stride(0) if l2 else 2
    check(L.rgsv_small_gsvd(pb1, ld1, l1, pb2, ld2, l2, n, vp(sv1), vp(sv2), vp(ints[0:2]),
                            vp(status), vp(ws), nb, st), "rgsv_small_gsvd")
    check(L.rgsv_comparative(vp(sv1), vp(ints[0:2]), vp(sv2), n, float(classify_tol),
                             *(vp(res[i * n:(i + 1) * n]) for i in range(6)),
                             vp(res[6 * n: 6 * n + 4]), vp(ints[2:4]), vp(status), st),
          "rgsv_comparative")
    h = res.cpu().numpy()
    iv = ints.cpu().numpy()
    names = ("alphas", "betas", "rho", "theta", "p1", "p2")
    out = {k: h[i * n:(i + 1) * n].copy() for i, k in enumerate(names)}
    out["scalars"] = h[6 * n: 6 * n + 4].copy()
    off = 6 * n + 4
    w = max(l1, l2, 1)
    out["sv1"] = h[off: off + int(iv[0])].copy()
    out["sv2"] = h[off + w: off + w + int(iv[1])].copy()
    out["counts"] = (int(iv[2]), int(iv[3]))
    out["status"] = int(iv[4])
    return out


# ----------------------------------------------------------------- results
class _Packed:
    """One device buffer + one pinned host mirror holding every small output
    of a pair, so a single D2H copy returns all of them."""

    def __init__(self, n: int, k1: int, k2: int):
        self.n = n
        f = [("stats1", 2), ("stats2", 2), ("scalars", 4), ("sv1", max(k1, 1)),
             ("sv2", max(k2, 1)), ("alphas", n), ("betas", n), ("rho", n), ("theta", n),
             ("p1", n), ("p2", n), ("rdiag1", max(k1, 1)), ("rdiag2", max(k2, 1))]
        ints = [("status", 1), ("nsv", 2), ("counts", 2)]
        self.off = {}
        pos = 0
        for name, cnt in f:
            self.off[name] = ("f", pos, cnt)
            pos += cnt * 8
        for name, cnt in ints:
            self.off[name] = ("i", pos, cnt)
            pos += cnt * 4
        self.nbytes = (pos + 15) // 16 * 16
        self.dev = torch.zeros(self.nbytes, dtype=torch.uint8, device="cuda")
        self.host = torch.zeros(self.nbytes, dtype=torch.uint8, pin_memory=True)
        self.hnp = self.host.numpy()

    def d(self, name) -> torch.Tensor:
        kind, pos, cnt = self.off[name]
        width = 8 if kind == "f" else 4
        view = self.dev[pos:pos + cnt * width]
        return view.view(F64 if kind == "f" else torch.int32)

    def h(self, name) -> np.ndarray:
        kind, pos, cnt = self.off[name]
        dt = np.float64 if kind == "f" else np.int32
        return self.hnp[pos:pos + cnt * (8 if kind == "f" else 4)].view(dt)


@dataclass
class MatrixOut:
    q: torch.Tensor      # m x kp (device)
    b: torch.Tensor      # kp x ldb (device)
    k: int


class SketchPlan:
    """Buffers for one matrix chain (m x n, rank k)."""

    def __init__(self, m: int, n: int, k: int):
        self.m, self.n, self.k = m, n, k
        self.kp = ceil16(k)
        self.ldb = ceil16(n)
        L = lib()
        self.ws_bytes = int(L.rgsv_sketch_workspace_bytes(m, n, k))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device="cuda")
        self.q = torch.zeros((m, self.kp), dtype=F64, device="cuda")
        self.b = torch.zeros((self.kp, self.ldb), dtype=F64, device="cuda")
        self.om_dev = torch.zeros((self.kp, self.ldb), dtype=F64, device="cuda")
        self.seed_host = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        self.seed_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.om_ws_bytes = int(L.rgsv_omega_workspace_bytes(1, n, k))
        self.om_ws = torch.empty(self.om_ws_bytes, dtype=torch.uint8, device="cuda")

    def set_seed(self, seed: int) -> None:
        """Host side of Omega: only the 8-byte seed (the H2D copy and the
        generation are part of the launch sequence / CUDA graph)."""
        self.seed_host[0] = seed_word(seed)

    def enqueue_omega(self, status: torch.Tensor, stream) -> None:
        """Omega^T for this chain, generated on the device (rgsv_omega_generate)."""
        with torch.cuda.stream(stream):
            self.seed_dev.copy_(self.seed_host, non_blocking=True)
        rc = lib().rgsv_omega_generate(vp(self.seed_dev), 1, self.n, self.k, vp(self.om_dev),
                                       self.ldb, 0, vp(status), vp(self.om_ws), self.om_ws_bytes,
                                       sp(stream))
        check(rc, "rgsv_omega_generate")

    def launch(self, g: DevMatrix, q_iters: int, stats: torch.Tensor, rdiag: torch.Tensor,
               status: torch.Tensor, stream) -> None:
        rc = lib().rgsv_sketch_project(
            vp(g.t), g.ld, g.rows, g.cols, vp(self.om_dev), self.ldb, self.k, q_iters,
            vp(self.q), vp(self.b), self.ldb, vp(stats), vp(rdiag), vp(status), vp(self.ws),
            self.ws_bytes, sp(stream))
        check(rc, "rgsv_sketch_project")


class PairPlan:
    """Cached buffers for a pair of shapes (m, p, n) at ranks (k1, k2)."""

    def __init__(self, m: int, p: int, n: int, k1: int, k2: int):
        self.m, self.p, self.n, self.k1, self.k2 = m, p, n, k1, k2
        self.s1 = SketchPlan(m, n, k1)
        self.s2 = SketchPlan(p, n, k2)
        self.small_bytes = int(lib().rgsv_small_gsvd_workspace_bytes(k1, k2, n))
        self.small_ws = torch.empty(self.small_bytes, dtype=torch.uint8, device="cuda")
        self.pk = _Packed(n, k1, k2)
        self.side = torch.cuda.Stream()
        self.graph = None
        self.graph_key = None
        self.last_key = None
        self.kernels_per_replay = 0

    def enqueue(self, g1: DevMatrix, g2: DevMatrix, q_iters: int, classify_tol: float,
                ready1=None, ready2=None) -> None:
        """Every device operation of one pair, on the current stream (G1
        chain, small GSVD, comparative kernel, packed D2H) and the side
        stream (G2 chain). Capturable as one CUDA graph. ready1 / ready2:
        optional events after which G1 / G2 are valid (the end-to-end path
        starts the G1 chain while G2 is still crossing PCIe)."""
        L = lib()
        main = torch.cuda.current_stream()
        pk = self.pk
        pk.d("status").zero_()
        self.side.wait_stream(main)
        self.s1.enqueue_omega(pk.d("status"), main)
        self.s2.enqueue_omega(pk.d("status"), self.side)
        if ready1 is not None:
            main.wait_event(ready1)
        if ready2 is not None:
            self.side.wait_event(ready2)
        self.s1.launch(g1, q_iters, pk.d("stats1"), pk.d("rdiag1"), pk.d("status"), main)
        self.s2.launch(g2, q_iters, pk.d("stats2"), pk.d("rdiag2"), pk.d("status"), self.side)
        main.wait_stream(self.side)
        rc = L.rgsv_small_gsvd(vp(self.s1.b), self.s1.ldb, self.k1, vp(self.s2.b), self.s2.ldb,
                               self.k2, self.n, vp(pk.d("sv1")), vp(pk.d("sv2")),
                               vp(pk.d("nsv")), vp(pk.d("status")), vp(self.small_ws),
                               self.small_bytes, sp(main))
        check(rc, "rgsv_small_gsvd")
        rc = L.rgsv_comparative(vp(pk.d("sv1")), vp(pk.d("nsv")), vp(pk.d("sv2")), self.n,
                                float(classify_tol), vp(pk.d("alphas")), vp(pk.d("betas")),
                                vp(pk.d("rho")), vp(pk.d("theta")), vp(pk.d("p1")),
                                vp(pk.d("p2")), vp(pk.d("scalars")), vp(pk.d("counts")),
                                vp(pk.d("status")), sp(main))
        check(rc, "rgsv_comparative")
        pk.host.copy_(pk.dev, non_blocking=True)

    def run(self, g1: DevMatrix, g2: DevMatrix, seed: int, q_iters: int, classify_tol: float,
            sync: bool = True):
        """One pair: stage the two seeds (reference convention: seed for G1,
        seed + 1 for G2, engine.py:252-253), then replay the captured CUDA
        graph when the device buffers are the captured ones, otherwise launch
        eagerly (and capture on the second sighting)."""
        self.s1.set_seed(seed)
        self.s2.set_seed(int(seed) + 1)
        key = (g1.t.data_ptr(), g1.ld, g1.rows, g2.t.data_ptr(), g2.ld, g2.rows, int(q_iters),
               float(classify_tol))
        if self.graph is not None and self.graph_key == key:
            self.graph.replay()
            GRAPH_REPLAYS[0] += 1
            GRAPH_REPLAYS[1] += self.kernels_per_replay
        elif USE_GRAPHS and self.last_key == key:
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            n0 = lib().rgsv_launch_count()
            with torch.cuda.graph(graph):
                self.enqueue(g1, g2, q_iters, classify_tol)
            self.kernels_per_replay = lib().rgsv_launch_count() - n0
            self.graph, self.graph_key = graph, key
            graph.replay()
            GRAPH_REPLAYS[0] += 1
            GRAPH_REPLAYS[1] += self.kernels_per_replay
        else:
            self.enqueue(g1, g2, q_iters, classify_tol)
        self.last_key = key
        if sync:
            torch.cuda.current_stream().synchronize()
        return self.pk


USE_GRAPHS = True
# [graph replays, library kernels executed by those replays] (the C-ABI
# launch counter only sees launches issued while capturing)
GRAPH_REPLAYS = [0, 0]


class BatchPlan:
    """B independent pairs of one shape processed concurrently: each pair's
    two chains run on their own streams, all captured in ONE CUDA graph, so
    the single-CTA latency steps of every chain overlap the other chains'
    GEMMs (the throughput mode of compute_gsv_batch / compare_batch)."""

    def __init__(self, B: int, m: int, p: int, n: int, k1: int, k2: int):
        self.plans = [PairPlan(m, p, n, k1, k2) for _ in range(B)]
        self.streams = [torch.cuda.Stream() for _ in range(B)]
        self.graph = None
        self.graph_key = None
        self.last_key = None
        self.kernels_per_replay = 0

    def enqueue(self, pairs, q_iters: int, classify_tol: float) -> None:
        cur = torch.cuda.current_stream()
        for plan, st, (g1, g2) in zip(self.plans, self.streams, pairs):
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                plan.enqueue(g1, g2, q_iters, classify_tol)
        for st in self.streams:
            cur.wait_stream(st)

    def run(self, pairs, seeds, q_iters: int, classify_tol: float, sync: bool = True):
        for plan, seed in zip(self.plans, seeds):
            plan.s1.set_seed(seed)
            plan.s2.set_seed(int(seed) + 1)
        key = tuple((g1.t.data_ptr(), g1.ld, g1.rows, g2.t.data_ptr(), g2.ld, g2.rows)
                    for g1, g2 in pairs) + (int(q_iters), float(classify_tol))
        if self.graph is not None and self.graph_key == key:
            self.graph.replay()
            GRAPH_REPLAYS[0] += 1
            GRAPH_REPLAYS[1] += self.kernels_per_replay
        elif USE_GRAPHS and self.last_key == key:
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            n0 = lib().rgsv_launch_count()
            with torch.cuda.graph(graph):
                self.enqueue(pairs, q_iters, classify_tol)
            self.kernels_per_replay = lib().rgsv_launch_count() - n0
            self.graph, self.graph_key = graph, key
            graph.replay()
            GRAPH_REPLAYS[0] += 1
            GRAPH_REPLAYS[1] += self.kernels_per_replay
        else:
            self.enqueue(pairs, q_iters, classify_tol)
        self.last_key = key
        if sync:
            torch.cuda.current_stream().synchronize()
        return [plan.pk for plan in self.plans]


class HostStreamPlan:
    """B pairs whose G1, G2 live in HOST memory (the end-to-end path): the
    H2D copies of every pair run back to back on one copy stream, and pair
    b's captured compute graph starts on its own stream as soon as pair b's
    copy event fires, so compute overlaps the transfers of the pairs behind
    it and the step is bounded by the PCIe link, not by copy + compute.
    Large pairs (>= BIG_PAIR_BYTES, e.g. the genome-scale cfg2) are enqueued
    eagerly with one event per matrix instead: the G1 chain runs while G2 is
    still being copied."""

    BIG_PAIR_BYTES = 1 << 30

    def __init__(self, B: int, m: int, p: int, n: int, k1: int, k2: int):
        self.B, self.m, self.p, self.n = B, m, p, n
        self.plans = [PairPlan(m, p, n, k1, k2) for _ in range(B)]
        self.streams = [torch.cuda.Stream() for _ in range(B)]
        self.copy_stream = torch.cuda.Stream()
        self.events = [torch.cuda.Event() for _ in range(B)]
        self.events1 = [torch.cuda.Event() for _ in range(B)]
        w = _even(n)
        self.bufs = []
        for _ in range(B):
            d1 = torch.zeros((m, w), dtype=F64, device="cuda")
            d2 = torch.zeros((p, w), dtype=F64, device="cuda")
            self.bufs.append((DevMatrix(d1[:, :n], m, n), DevMatrix(d2[:, :n], p, n)))

    @staticmethod
    def _host(a, rows, cols, name):
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a))
        if t.dim() != 2 or tuple(t.shape) != (rows, cols):
            raise DimensionError(f"{name}: expected shape {(rows, cols)}, got {tuple(t.shape)}")
        if t.is_complex():
            raise ValidationError(f"{name}: complex matrices are not supported by the B200 path")
        if t.dtype != F64:
            t = t.to(F64)
        if not t.is_contiguous():
            t = t.contiguous()
        if not t.is_pinned():
            t = t.pin_memory()  # async H2D needs page-locked memory
        return t

    def run(self, host_pairs, seeds, q_iters: int, classify_tol: float):
        cur = torch.cuda.current_stream()
        self.copy_stream.wait_stream(cur)
        staged = [(self._host(h1, self.m, self.n, "g1"), self._host(h2, self.p, self.n, "g2"))
                  for h1, h2 in host_pairs]
        big = 8 * (self.m + self.p) * self.n >= self.BIG_PAIR_BYTES
        with torch.cuda.stream(self.copy_stream):
            for (h1, h2), (d1, d2), ev1, ev in zip(staged, self.bufs, self.events1, self.events):
                d1.t.copy_(h1, non_blocking=True)
                ev1.record(self.copy_stream)
                d2.t.copy_(h2, non_blocking=True)
                ev.record(self.copy_stream)
        for plan, st, ev1, ev, (d1, d2), seed in zip(self.plans, self.streams, self.events1,
                                                      self.events, self.bufs, seeds):
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                if big:  # per-matrix readiness: chain 1 overlaps the G2 copy
                    plan.s1.set_seed(seed)
                    plan.s2.set_seed(int(seed) + 1)
                    plan.enqueue(d1, d2, q_iters, classify_tol, ready1=ev1, ready2=ev)
                else:
                    st.wait_event(ev)
                    plan.run(d1, d2, seed, q_iters, classify_tol, sync=False)
        for st in self.streams:
            cur.wait_stream(st)
        cur.synchronize()  # the pinned staging (if any) is released only after this
        return [plan.pk for plan in self.plans]


_HOST_PLANS: dict = {}


def host_stream_plan(B: int, m: int, p: int, n: int, k1: int, k2: int) -> HostStreamPlan:
    key = (torch.cuda.current_device(), B, m, p, n, k1, k2)
    plan = _HOST_PLANS.get(key)
    if plan is None:
        if len(_HOST_PLANS) > 2:
            _HOST_PLANS.clear()
        plan = HostStreamPlan(B, m, p, n, k1, k2)
        _HOST_PLANS[key] = plan
    return plan


_BATCH_PLANS: dict = {}


def batch_plan(B: int, m: int, p: int, n: int, k1: int, k2: int) -> BatchPlan:
    key = (torch.cuda.current_device(), B, m, p, n, k1, k2)
    plan = _BATCH_PLANS.get(key)
    if plan is None:
        if len(_BATCH_PLANS) > 4:
            _BATCH_PLANS.clear()
        plan = BatchPlan(B, m, p, n, k1, k2)
        _BATCH_PLANS[key] = plan
    return plan


_PLANS: dict = {}


def pair_plan(m: int, p: int, n: int, k1: int, k2: int) -> PairPlan:
    key = (torch.cuda.current_device(), m, p, n, k1, k2)
    plan = _PLANS.get(key)
    if plan is None:
        if len(_PLANS) > 8:
            _PLANS.clear()
        plan = PairPlan(m, p, n, k1, k2)
        _PLANS[key] = plan
    return plan


def residual_history(gf2: float, energy: float) -> list:
    """[||G||_F, sqrt(max(||G||^2 - captured, 0))] (rangefinder.py:94,126-127)."""
    return [math.sqrt(gf2), math.sqrt(max(gf2 - energy, 0.0))]


STAGE_BYTES = 2 << 30  # fp64 staging for streamed fp32 row chunks


def f64_chunks(g: DevMatrix, rows: int | None = None):
    """Yield (r0, r1, DevMatrix) fp64 row blocks of g: views for fp64 input,
    rgsv_convert_f32 promotions into one reused staging buffer for fp32."""
    if not g.is_f32:
        yield 0, g.rows, g
        return
    w = _even(g.cols)
    R = rows or max(64, min(g.rows, STAGE_BYTES // (8 * w)))
    stage = torch.zeros((min(R, g.rows), w), dtype=F64, device="cuda")
    st = sp(torch.cuda.current_stream())
    for r0 in range(0, g.rows, R):
        r1 = min(g.rows, r0 + R)
        check(lib().rgsv_convert_f32(ctypes.c_void_p(g.t.data_ptr() + r0 * g.ld * 4), g.ld,
                                     r1 - r0, g.cols, vp(stage), w, st), "rgsv_convert_f32")
        yield r0, r1, DevMatrix(stage[: r1 - r0, : g.cols], r1 - r0, g.cols)


def device_sumsq(g: DevMatrix) -> float:
    """||G||_F^2 on the device (core.sum_sq, core.py:115-125); fp32 input is
    promoted chunk by chunk (squares of fp32 values are exact in fp64)."""
    if g.is_f32:
        return math.fsum(device_sumsq(c) for _, _, c in f64_chunks(g))
    out = torch.zeros(1, dtype=F64, device="cuda")
    ws = torch.empty(1024, dtype=F64, device="cuda")
    rc = lib().rgsv_sumsq(vp(g.t), g.ld, g.rows, g.cols, vp(out), vp(ws), ws.numel() * 8,
                          sp(torch.cuda.current_stream()))
    check(rc, "rgsv_sumsq")
    return float(out.item())


__all__ = ["DevMatrix", "to_device", "pair_plan", "PairPlan", "SketchPlan", "omega_device",
           "residual_history", "device_sumsq", "ceil16", "_native"]


# ------------------------------------------------------- many small pairs
_DESC = np.dtype([("g", "<u8"), ("ld", "<i8"), ("rows", "<i4"), ("pad", "<i4")])


def small_batch_fits(max_rows: int, n: int, k1: int, k2: int) -> bool:
    """Shapes served by rgsv_batch_gsvd (the cfg3 kernels)."""
    return k1 == k2 and bool(lib().rgsv_batch_supported(max_rows, n, k1))


class SmallBatchPlan:
    """rgsv_batch_gsvd for B same-shape small pairs: descriptors, workspace
    and outputs live in HBM across calls; one packed D2H per run."""

    def __init__(self, B: int, n: int, k: int):
        require_device()
        self.B, self.n, self.k = B, n, k
        L = lib()
        self.ws_bytes = int(L.rgsv_batch_workspace_bytes(B, n, k))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device="cuda")
        self.res_stride = 6 * n + 4 + 2 * k
        # res | stats, one float64 buffer; ints | status, one int32 buffer
        self.fbuf = torch.zeros(B * self.res_stride + 4 * B, dtype=F64, device="cuda")
        self.ibuf = torch.zeros(5 * B, dtype=torch.int32, device="cuda")
        self.fhost = torch.empty(self.fbuf.shape, dtype=F64, pin_memory=True)
        self.ihost = torch.empty(self.ibuf.shape, dtype=torch.int32, pin_memory=True)
        self.desc = torch.zeros(2 * B * _DESC.itemsize, dtype=torch.uint8, device="cuda")
        self.seeds = torch.zeros(2 * B, dtype=torch.int64, device="cuda")
        self._desc_key = None
        self._pairs_key = None
        self._seed_key = None

    def set_pairs(self, pairs, key=None) -> int:
        """Descriptors {G1_j, G2_j} of the (resident) pairs; returns max rows.
        Cached on the identity of the matrix objects (kept referenced here so
        the identities stay valid while cached). `key`: an identity key the
        caller already holds for this very sequence (engine._batch_scan's
        tuple of pair ids) -- a hit then costs one tuple comparison instead of
        rebuilding the 2B-entry matrix list."""
        if key is not None and key == self._pairs_key:
            return self.max_rows
        mats = [g for pair in pairs for g in pair]
        mkey = tuple(map(id, mats))
        if mkey != self._desc_key:
            arr = np.zeros(len(mats), dtype=_DESC)
            arr["g"] = [g.t.data_ptr() for g in mats]
            arr["ld"] = [g.ld for g in mats]
            arr["rows"] = [g.rows for g in mats]
            self.desc.copy_(torch.from_numpy(arr.view(np.uint8)))
            self._desc_key = mkey
            self._desc_refs = mats
            self.max_rows = int(arr["rows"].max())
        self._pairs_key = key
        self._pairs_refs = pairs if key is not None else None  # keeps the keyed ids valid
        return self.max_rows

    def set_seeds(self, seeds) -> None:
        """Omega stream seeds: G1_j from seeds[j], G2_j from seeds[j] + 1
        (engine.py:252-253), reduced mod 2^64 like rangefinder.py:101."""
        try:  # one vectorized conversion when every seed fits int64 (the usual case)
            sd = np.asarray(seeds, dtype=np.int64).astype(np.uint64)  # two's complement = mod 2^64
            if sd.ndim != 1:
                raise TypeError
        except (OverflowError, TypeError, ValueError):
            sd = np.fromiter((int(x) & SEED_MASK for x in seeds), dtype=np.uint64,
                             count=len(seeds))
        words = np.empty(2 * len(sd), dtype=np.uint64)
        words[0::2] = sd
        words[1::2] = sd + np.uint64(1)  # wraps mod 2^64
        self.seeds.copy_(torch.from_numpy(words.view(np.int64)))

    def launch(self, q_iters: int, classify_tol: float, stream=None, b_out=None) -> None:
        """b_out: optional (2B x kp x ceil16(n)) tensor receiving every B."""
        st = stream or torch.cuda.current_stream()
        B, n, k = self.B, self.n, self.k
        res = self.fbuf[: B * self.res_stride]
        stats = self.fbuf[B * self.res_stride:]
        bo = vp(b_out) if b_out is not None else ctypes.c_void_p(0)
        check(lib().rgsv_batch_gsvd(vp(self.desc), B, self.max_rows, n, k, q_iters,
                                    vp(self.seeds), float(classify_tol), vp(res),
                                    vp(self.ibuf[: 4 * B]), vp(stats), vp(self.ibuf[4 * B:]), bo,
                                    vp(self.ws), self.ws_bytes, sp(st)), "rgsv_batch_gsvd")

    def fetch(self):
        """One packed D2H of the results into FRESH pinned buffers (torch's
        caching host allocator recycles them once the caller drops the
        previous results), returned as numpy views: nothing is copied on the
        host, and earlier results stay valid."""
        fh = torch.empty(self.fbuf.shape, dtype=F64, pin_memory=True)
        ih = torch.empty(self.ibuf.shape, dtype=torch.int32, pin_memory=True)
        fh.copy_(self.fbuf, non_blocking=True)
        ih.copy_(self.ibuf, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return fh.numpy(), ih.numpy()

    def run(self, pairs, seeds, q_iters: int, classify_tol: float, key=None):
        self.set_pairs(pairs, key)
        self.set_seeds(seeds)
        self.launch(q_iters, classify_tol)
        return self.fetch()


_SMALL_PLANS: dict = {}


def small_batch_plan(B: int, n: int, k: int) -> SmallBatchPlan:
    key = (torch.cuda.current_device(), B, n, k)
    plan = _SMALL_PLANS.get(key)
    if plan is None:
        if len(_SMALL_PLANS) > 4:
            _SMALL_PLANS.clear()
        plan = SmallBatchPlan(B, n, k)
        _SMALL_PLANS[key] = plan
    return plan
