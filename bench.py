#!/usr/bin/env python
"""rGSVD benchmark: pairs/s and sketch-GEMM TFLOP/s on B200.

    python bench.py [--gpus N --steps K --warmup W] [--config cfg1] [--impl reference]

A step is one full randomized GSVD + comparative analysis of a batch of B
independent matrix pairs (BASELINE.json configs) run concurrently through
compare_batch, with fresh Ω seeds every step (the reference's run_bench
convention, bench.py:98-102). The default workload is cfg2, the config
BASELINE.json's metric is quoted on ("Throughput reported at 1/2/4/8
GPUs"): fp64, m=200000, p=150000, n=4000, k=120, q=2, one pair per step.
latency_ms_per_pair reports one pair at a time through compare(). Synthetic seeded data with the
config's shape/rank/noise (paper_2404_09459_b200/workloads.py) stands in
for the paper's genome datasets.

value  : pairs/s with all G resident in HBM (whole job = all ranks).
e2e    : the same through the public API with G1, G2 in pinned HOST
         memory: every step copies them H2D and reads the report D2H.
roofline: the dominant GEMM kernel timed live with CUDA events on its
         stream; algorithmic flops 2 m n k per launch; peak = FP64 DMMA
         issue peak measured on this pool (profiles/r01_fp64_peak.log).
cpu_baseline: the CPU oracle (numpy restatement of the reference with the
         q power iterations; OpenBLAS on the host cores) on a bounded sample.
N > 1 : one process per GPU. Single-pair configs (cfg2, cfg4; cfg0/cfg1
         with --sharded) run ONE pair per step row-sharded over the ranks
         (dist.py: NCCL all-reduce of the Gram / Z / B partials), "strong"
         scaling, as north_star asks; --replicas times independent replica
         pairs per rank instead ("weak"). cfg3 is always replicas (its pairs
         are independent).
metric: the same string in both arms ("rGSVD pairs/sec (cfgN)"), so the
         driver can pair our line with the reference arm's; the sketch-GEMM
         TFLOP/s and its roofline fraction are separate keys.
cfg4   : fp32 pairs run the G passes on the tcgen05 tensor cores (3xTF32);
         the roofline is against 3xTF32 = measured bf16 burst / 2 / 3.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 37.0  # tools/fp64_peak.cu on this pool's B200 (profiles/r01_fp64_peak.log)


def _measured_bf16() -> float:
    """bf16 burst TFLOP/s from the driver-written MEASURED_PEAKS.json
    (fallback: the profiling recipe's 1.59 PFLOP/s)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return 1590.0


MEASURED_BF16_TFLOPS = _measured_bf16()


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--batch", type=int, default=None,
                    help="independent pairs per step, processed concurrently (compare_batch); "
                         "default 8 for cfg0/cfg1 (measured 643/676/686 pairs/s at 4/6/8 on "
                         "cfg1), 1 for the genome-scale cfg2, "
                         "the config's batch for cfg3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="ONE pair row-sharded over the ranks (dist.compute_gsv_sharded, NCCL "
                         "all-reduce of the Gram / Z / B partials): strong scaling; the default "
                         "at N > 1 for the single-pair configs")
    ap.add_argument("--replicas", action="store_true",
                    help="at N > 1: independent replica pairs per rank (weak scaling) instead "
                         "of one row-sharded pair")
    return ap.parse_args()


def metric(cfg) -> str:
    """The metric string both arms print (identical, so the driver pairs them)."""
    return f"rGSVD pairs/sec ({cfg.name})"


class Clocks:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.rows = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, smax, reasons = [], None, set()
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
            except ValueError:
                continue
            for name, val in zip(names, r[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(cfg, budget_s: float, g1, g2):
    """Oracle restatement on the host cores, bounded sample of whole pairs."""
    from oracle import rgsv_oracle as orc

    threads = _all_blas_threads()
    t_start = time.perf_counter()
    done = 0
    while True:
        orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=done)
        done += 1
        if time.perf_counter() - t_start > budget_s or done >= 50:
            break
    dt = time.perf_counter() - t_start
    return {"value": done / dt, "unit": "pairs/s", "cores": threads, "kind": "port",
            "sample": f"{done} whole {cfg.name} pairs (k={cfg.k}, q={cfg.q}) through "
                      f"oracle/rgsv_oracle.run_pipeline, numpy {__import__('numpy').__version__}"
                      f" + OpenBLAS on {threads} host threads, {dt:.1f} s"}


def workload_desc(cfg):
    """The workload string both arms print (config.workload)."""
    seeds = "per-pair Omega seeds 2j, 2j+1" if cfg.batch > 1 else "Omega seed = step index"
    return (f"{cfg.name}: {cfg.dtype} rGSVD pair m={cfg.m} p={cfg.p} n={cfg.n} s={cfg.s} "
            f"(shared {cfg.shared}) decay 10^(-{cfg.decay:g} j/s) eps={cfg.eps:g} k={cfg.k} "
            f"q={cfg.q}, fixed-rank range finder, {seeds}")


def _all_blas_threads() -> int:
    """Let the host BLAS use every core (torchrun exports OMP_NUM_THREADS=1
    to its workers); returns the thread count in effect."""
    n = os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_info, threadpool_limits

        threadpool_limits(limits=n, user_api="blas")
        got = [p.get("num_threads", n) for p in threadpool_info() if p.get("user_api") == "blas"]
        return max(got) if got else n
    except Exception:  # threadpoolctl missing: report the env setting
        return int(os.environ.get("OPENBLAS_NUM_THREADS", os.environ.get("OMP_NUM_THREADS", n)))


def run_reference(args, rank, world):
    """The reference arm: the CPU restatement of the reference path
    (oracle/rgsv_oracle.run_pipeline: bench._timed_run's region, reference
    bench.py:72-79, plus the q power iterations the reference lacks) on the
    same config, whole pairs per step, all host cores. Rank 0 only."""
    from paper_2404_09459_b200.workloads import CONFIGS, make_pair

    if rank != 0:
        return
    threads = _all_blas_threads()
    cfg = CONFIGS[args.config]
    scale, inst = 1.0, ""
    if cfg.dtype == "f32":  # cfg4: 118 GB of host fp64; a 1/50-row instance, scaled by rows
        ms, ps = cfg.m // 50, cfg.p // 50
        g1, g2 = make_pair(cfg, m=ms, p=ps)
        scale = (ms + ps) / (cfg.m + cfg.p)
        inst = (f"; each step one m={ms} p={ps} instance (1/50 of the rows, fp64 as the reference "
                f"promotes), pairs/s scaled by rows x{scale:.4f}")
    else:
        g1, g2 = make_pair(cfg)
    from oracle import rgsv_oracle as orc

    for i in range(args.warmup):
        orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        orc.run_pipeline(g1, g2, k=cfg.k, q=cfg.q, seed=i)
    dt = time.perf_counter() - t0
    value = args.steps / dt * scale
    line = {
        "impl": "reference", "metric": metric(cfg), "value": value,
        "unit": "pairs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(cfg), "g_bytes": cfg.g_bytes,
                   "parallelism": "host cores"},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{args.steps} whole pairs through the numpy restatement of "
                                   "the reference (oracle/rgsv_oracle.py; the reference has no "
                                   f"power iteration, SURVEY.md §0 F1), OpenBLAS on {threads} "
                                   f"host threads{inst}"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def committed_traffic(cfg_name: str, kernel: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
    of `kernel` at this config's shapes, from the newest committed ncu
    summary profiles/rNN_gemm_<cfg>_traffic.json (None when there is none)."""
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_*{cfg_name}_traffic.json")),
                       reverse=True):
        try:
            d = json.load(open(path)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            continue
        if isinstance(d, dict):
            if kernel in d:
                return float(d[kernel])
        elif d is not None and kernel == "k_gtq":  # round-1 format: the gtq launch only
            return float(d)
    return None


def time_kernel(fn, reps=20):
    import torch

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def device_batch_pairs(cfg, B, seed0):
    """cfg3-style batch generated on the device with the workloads.py
    recipe (G_i = (A_i diag d) B_i^T + eps E_i, B2 sharing B1's first
    `shared` columns), seeded per rank; returns (g1, g2) as (B, rows, n)."""
    import torch

    gen = torch.Generator(device="cuda").manual_seed(seed0)
    f64 = torch.float64
    a1 = torch.randn((B, cfg.m, cfg.s), generator=gen, device="cuda", dtype=f64)
    a2 = torch.randn((B, cfg.p, cfg.s), generator=gen, device="cuda", dtype=f64)
    b1 = torch.randn((B, cfg.n, cfg.s), generator=gen, device="cuda", dtype=f64)
    b2 = torch.cat([b1[:, :, : cfg.shared],
                    torch.randn((B, cfg.n, cfg.s - cfg.shared), generator=gen, device="cuda",
                                dtype=f64)], dim=2)
    d = 10.0 ** (-cfg.decay * torch.arange(cfg.s, device="cuda", dtype=f64) / cfg.s)
    g1 = torch.bmm(a1 * d, b1.transpose(1, 2))
    g1 += cfg.eps * torch.randn(g1.shape, generator=gen, device="cuda", dtype=f64)
    g2 = torch.bmm(a2 * d, b2.transpose(1, 2))
    g2 += cfg.eps * torch.randn(g2.shape, generator=gen, device="cuda", dtype=f64)
    return g1, g2


def run_ours_batch(args, rank, world):
    """cfg3: every step is compare_batch over all cfg.batch pairs (one
    rgsv_batch_gsvd call: Omega for every matrix, one clustered chain launch,
    one small-GSVD launch)."""
    import torch
    import torch.distributed as dist

    import paper_2404_09459_b200 as rg
    from paper_2404_09459_b200 import _native
    from paper_2404_09459_b200 import device as dv
    from paper_2404_09459_b200.workloads import CONFIGS, make_pair

    cfg = CONFIGS[args.config]
    B = cfg.batch if args.batch in (None, 0) else args.batch
    g1, g2 = device_batch_pairs(cfg, B, 1000 + rank)
    pairs = [rg.GmpPair.resident(g1[j], g2[j]) for j in range(B)]
    base = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step(i):  # per-pair Omega seeds 2j (+1 for G2), shifted every step
        return rg.compare_batch(pairs, base, seeds=[2 * (i * B + j) for j in range(B)])

    for i in range(args.warmup):
        step(i)
    barrier()
    clocks = Clocks(torch.cuda.current_device()) if rank == 0 else None
    l0 = _native.lib().rgsv_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        reps = step(i)
    e1.record(stream)
    barrier()
    launches = _native.lib().rgsv_launch_count() - l0
    t = e0.elapsed_time(e1) * 1e-3
    clk = clocks.stop() if clocks else None
    tt = torch.tensor([t], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max = float(tt.item())
    value = args.steps * B * world / t_max

    # device-only batch call (no host unpacking), timed live on its stream
    plan = dv.small_batch_plan(B, cfg.n, cfg.k)
    plan.set_pairs([(pr.g1, pr.g2) for pr in pairs])
    plan.set_seeds([2 * j for j in range(B)])
    t_call = time_kernel(lambda: plan.launch(cfg.q, base.classify_tol), reps=5)
    flop = cfg.flops * B
    achieved = flop / t_call / 1e12

    # e2e: the same public call with the pairs in pinned host memory (a
    # bounded slice of the batch so the host buffers stay small)
    Be = min(B, 512)
    h1 = g1[:Be].cpu().pin_memory()
    h2 = g2[:Be].cpu().pin_memory()
    d1 = torch.empty_like(h1, device="cuda")
    d2 = torch.empty_like(h2, device="cuda")

    def e2e_step(i):
        d1.copy_(h1, non_blocking=True)
        d2.copy_(h2, non_blocking=True)
        prs = [rg.GmpPair.resident(d1[j], d2[j]) for j in range(Be)]
        return rg.compare_batch(prs, base, seeds=[2 * (i * Be + j) for j in range(Be)])

    for i in range(2):
        e2e_step(i)
    barrier()
    e0.record(stream)
    ne = max(3, args.steps)
    for i in range(ne):
        e2e_step(i)
    e1.record(stream)
    barrier()
    e2e_value = ne * Be * world / (e0.elapsed_time(e1) * 1e-3)
    eplan = dv.small_batch_plan(Be, cfg.n, cfg.k)
    h2d = h1.numel() * 8 + h2.numel() * 8 + 2 * Be * 8
    d2h = eplan.fhost.numel() * 8 + eplan.ihost.numel() * 4

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # N=1 only (contract)
        hg1, hg2 = make_pair(cfg, data_seed=0)
        cpu = cpu_baseline(cfg, args.cpu_sample_seconds, hg1, hg2)
    if rank == 0:
        rep = reps[0]
        line = {
            "metric": metric(cfg),
            "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated with the workloads.py recipe)",
            "config": {"workload": workload_desc(cfg),
                       "batch": B, "g_bytes_total": cfg.g_bytes * B,
                       "l2": "inputs larger than L2 (%.1f GB > 126 MB)" % (cfg.g_bytes * B / 1e9),
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
            "roofline": {"bound": "tensor", "kernel": "rgsv_batch_gsvd (k_batch_chain dominant)",
                         "achieved": achieved, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_DMMA_PEAK_TFLOPS, "traffic": None,
                         "flop_per_launch": flop, "launch_us": t_call * 1e6,
                         "hbm_4pass_equiv_GBps": cfg.stream_bytes * B / t_call / 1e9,
                         "note": "G is read from HBM once per chain (cluster re-reads hit L2); "
                                 "the 4-pass byte model of SURVEY.md §8 is reported for "
                                 "comparison"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "batch": Be,
                    "path": f"compare_batch() over {Be} pairs copied from pinned host memory "
                            "every step"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "check": {"r": int(rep.spectrum.r), "s": int(rep.spectrum.s), "d1": rep.d1,
                      "d2": rep.d2},
        }
        print(json.dumps(line), flush=True)


def device_f32_matrix(rows, cfg, a_seed, bmat, d):
    """fp32 G = (A diag d) B^T + eps E generated on the device in row chunks."""
    import torch

    torch.backends.cuda.matmul.allow_tf32 = False
    gen = torch.Generator(device="cuda").manual_seed(a_seed)
    g = torch.empty((rows, cfg.n), dtype=torch.float32, device="cuda")
    R = 1 << 16
    for r0 in range(0, rows, R):
        r1 = min(rows, r0 + R)
        a = torch.randn((r1 - r0, cfg.s), generator=gen, device="cuda", dtype=torch.float32)
        g[r0:r1] = (a * d) @ bmat.T
        g[r0:r1] += cfg.eps * torch.randn((r1 - r0, cfg.n), generator=gen, device="cuda",
                                          dtype=torch.float32)
    return g


def run_ours_f32(args, rank, world):
    """cfg4: one fp32-resident pair per step (59 GB in HBM). The four G
    passes per matrix run on the tcgen05 tensor cores as 3xTF32 GEMMs
    (fp32-level accuracy, csrc/tf32x3.cu); the small factorizations stay
    fp64 (DMMA). The reference promotes fp32 input to fp64 (core.py:51-54);
    GsvOptions(f32_mode="promote") reproduces that on the device."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2404_09459_b200 as rg
    from paper_2404_09459_b200 import _native
    from paper_2404_09459_b200 import device as dv
    from paper_2404_09459_b200.workloads import CONFIGS, make_pair

    cfg = CONFIGS[args.config]
    gen = torch.Generator(device="cuda").manual_seed(77 + rank)
    b1 = torch.randn((cfg.n, cfg.s), generator=gen, device="cuda", dtype=torch.float32)
    b2 = torch.cat([b1[:, : cfg.shared],
                    torch.randn((cfg.n, cfg.s - cfg.shared), generator=gen, device="cuda",
                                dtype=torch.float32)], dim=1)
    d = (10.0 ** (-cfg.decay * torch.arange(cfg.s, device="cuda", dtype=torch.float64)
                  / cfg.s)).float()
    g1 = device_f32_matrix(cfg.m, cfg, 1000 + rank, b1, d)
    g2 = device_f32_matrix(cfg.p, cfg, 2000 + rank, b2, d)
    pair = rg.GmpPair.resident(g1, g2)
    stream = torch.cuda.current_stream()

    def opts(seed):
        return rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, seed, cfg.q))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        rg.compare(pair, opts(i))
    barrier()
    clocks = Clocks(torch.cuda.current_device()) if rank == 0 else None
    l0 = _native.lib().rgsv_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        rep = rg.compare(pair, opts(i))
    e1.record(stream)
    barrier()
    launches = _native.lib().rgsv_launch_count() - l0
    t = e0.elapsed_time(e1) * 1e-3
    clk = clocks.stop() if clocks else None
    tt = torch.tensor([t], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max = float(tt.item())
    value = args.steps * world / t_max

    # dominant kernels: the two 3xTF32 tcgen05 GEMM passes over all of G1,
    # timed live with CUDA events on their stream
    from paper_2404_09459_b200 import tf32 as tf

    kp, ldn = dv.ceil16(cfg.k), dv.ceil16(cfg.n)
    kq = (kp + 31) // 32 * 32
    ops = tf.TF32Ops()
    gm = dv.to_device(g1, "g1", keep_f32=True)
    lo, _ = ops.split_big(gm)
    xt = torch.zeros((kp, ldn), dtype=torch.float64, device="cuda")
    xt[: cfg.k, : cfg.n] = torch.randn(cfg.k, cfg.n, dtype=torch.float64, device="cuda")
    xh, xl = ops.split_small(xt, kp, ldn, ldn, rows_out=kq)
    Y = torch.empty((cfg.m, kq), dtype=torch.float64, device="cuda")
    qh, ql = ops.split_small(torch.randn(cfg.m, kq, dtype=torch.float64, device="cuda"),
                             cfg.m, kq, kq)
    Z = torch.zeros((kq, ldn), dtype=torch.float64, device="cuda")

    def gx():
        ops.gx(gm, lo, xh, xl, Y, cfg.m, kq, cfg.n)

    def gtq():
        ops.gtq(qh, ql, gm, lo, Z, kq, cfg.n, cfg.m)

    def split():
        ops.split_big(gm, lo)

    gtq()
    t_gx = time_kernel(gx, reps=5)
    t_gtq = time_kernel(gtq, reps=5)
    t_split = time_kernel(split, reps=5)
    flop = 2.0 * cfg.m * cfg.n * cfg.k          # algorithmic (k real columns)
    ach_gx, ach_gtq = flop / t_gx / 1e12, flop / t_gtq / 1e12
    # per pair: 2q+2 passes per matrix at the two kernels' rates (sketch +
    # q G*Qhat are gx; q G^T Q + projection are gtq)
    est = (cfg.q + 1) * (cfg.m + cfg.p) / cfg.m * (t_gx + t_gtq)
    share = est / (t_max / args.steps)
    tf32_peak = MEASURED_BF16_TFLOPS / 2.0      # TF32 dense = half the bf16 rate
    peak3 = tf32_peak / 3.0                     # 3 TF32 MMAs per fp32-accurate product
    dom_gx = t_gx * 1.0 <= t_gtq * 1.0
    achieved = ach_gtq if dom_gx else ach_gx
    del Y, qh, ql, Z, lo

    # e2e: the public call from pinned host fp32 arrays, on a 1/10-row
    # instance (the full 59 GB pair would not fit pinned host memory)
    me, pe = cfg.m // 10, cfg.p // 10
    h1 = g1[:me].cpu().pin_memory()
    h2 = g2[:pe].cpu().pin_memory()
    rg.compare(rg.GmpPair(h1, h2, check_rank=False), opts(0))
    torch.cuda.synchronize()
    e0.record(stream)
    ne = 3
    for i in range(ne):
        rep_e = rg.compare(rg.GmpPair(h1, h2, check_rank=False), opts(i))
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_value = ne / (e0.elapsed_time(e1) * 1e-3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # N=1 only (contract)
        # oracle on a 1/50-row fp64 instance, extrapolated linearly in rows
        ms, ps = cfg.m // 50, cfg.p // 50
        hg1, hg2 = make_pair(cfg, data_seed=0, m=ms, p=ps)
        sub = cpu_baseline(cfg, args.cpu_sample_seconds, hg1, hg2)
        scale = (ms + ps) / (cfg.m + cfg.p)
        cpu = {"value": sub["value"] * scale, "unit": "pairs/s", "cores": sub["cores"],
               "kind": "port",
               "sample": f"{sub['sample']}; instance m={ms}, p={ps} (1/50 of the rows, fp64 as "
                         f"the reference promotes), {sub['value']:.3f} pairs/s on it, scaled by "
                         f"rows {scale:.4f} (the work is linear in m+p); the full pair needs "
                         "118 GB of host fp64"}
    if rank == 0:
        line = {
            "metric": metric(cfg),
            "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 (3xTF32 tensor-core GEMMs, fp64 small factorizations)",
            "data": "synthetic (device-generated fp32 with the workloads.py recipe)",
            "config": {"workload": workload_desc(cfg), "g_bytes": cfg.g_bytes,
                       "l2": "inputs larger than L2 (%.1f GB)" % (cfg.g_bytes / 1e9),
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
            "roofline": {"bound": "tensor",
                         "kernel": ("tf32x3_gtq (Q^T G, split-K)" if dom_gx else
                                    "tf32x3_gx (G X^T)") + " over G1 (m x n)",
                         "achieved": achieved, "peak": peak3, "unit": "TFLOP/s",
                         "frac": achieved / peak3, "traffic": None,
                         "peak_source": "3xTF32: measured bf16 burst (MEASURED_PEAKS.json "
                                        f"{MEASURED_BF16_TFLOPS}) / 2 for TF32 / 3 MMAs per "
                                        "fp32-accurate product",
                         "flop_per_launch": flop,
                         "launch_us": {"tf32x3_gx": t_gx * 1e6, "tf32x3_gtq": t_gtq * 1e6,
                                       "f32_split": t_split * 1e6},
                         "tflops": {"tf32x3_gx": ach_gx, "tf32x3_gtq": ach_gtq},
                         "gemm_share_of_step_est": share},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "pairs/s",
                    "h2d_bytes_per_step": int(h1.numel() * 4 + h2.numel() * 4),
                    "d2h_bytes_per_step": int((6 * cfg.n + 8) * 8),
                    "instance": f"m={me}, p={pe} (1/10 of the rows), fp32 pinned host arrays "
                                "through GmpPair + compare()"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "check": {"r": int(rep.spectrum.r), "s": int(rep.spectrum.s), "d1": rep.d1,
                      "d2": rep.d2},
        }
        print(json.dumps(line), flush=True)


def device_matrix(rows, cfg, a_seed, bmat, d, dtype):
    """G = (A diag d) B^T + eps E generated on the device in row chunks."""
    import torch

    torch.backends.cuda.matmul.allow_tf32 = False
    gen = torch.Generator(device="cuda").manual_seed(a_seed)
    g = torch.empty((rows, cfg.n), dtype=dtype, device="cuda")
    R = 1 << 15
    for r0 in range(0, rows, R):
        r1 = min(rows, r0 + R)
        a = torch.randn((r1 - r0, cfg.s), generator=gen, device="cuda", dtype=dtype)
        g[r0:r1] = (a * d) @ bmat.T
        g[r0:r1] += cfg.eps * torch.randn((r1 - r0, cfg.n), generator=gen, device="cuda",
                                          dtype=dtype)
    return g


def fp64_gemm_roofline(cfg, gmat, rows: int, steps_time_per_pair: float, world: int = 1):
    """Time the two G-pass DMMA GEMMs (B = Q^T G and Y = G X) live on G's
    shape (rows x n) with CUDA events on their stream; the slower one is the
    roofline kernel. Returns (roofline dict, sketch-GEMM TFLOP/s, kernel_us)."""
    import torch

    from paper_2404_09459_b200 import _native
    from paper_2404_09459_b200 import device as dv

    L = _native.lib()
    kp, ldb = dv.ceil16(cfg.k), dv.ceil16(cfg.n)
    Q = torch.randn(rows, kp, dtype=torch.float64, device="cuda")
    Q[:, cfg.k:] = 0
    Bo = torch.zeros(kp, ldb, dtype=torch.float64, device="cuda")
    Xt = torch.zeros(kp, ldb, dtype=torch.float64, device="cuda")
    Xt[: cfg.k, : cfg.n] = torch.randn(cfg.k, cfg.n, dtype=torch.float64, device="cuda")
    Y = torch.zeros(rows, kp, dtype=torch.float64, device="cuda")
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = dv.sp(torch.cuda.current_stream())

    # the chain runs the exact-width (120-wide) tiles when k = 120 (cfg2):
    # time the same kernels by asking for exactly the live width
    kl = cfg.k if cfg.k == 120 else kp

    def gtq():
        L.rgsv_gemm_gtq(dv.vp(Q), kp, dv.vp(gmat.t), gmat.ld, dv.vp(Bo), ldb, kl, cfg.n, rows,
                        dv.vp(scratch), scratch.numel(), st)

    def gx():
        L.rgsv_gemm_gx(dv.vp(gmat.t), gmat.ld, dv.vp(Xt), ldb, dv.vp(Y), kp, rows, kl, cfg.n,
                       dv.vp(scratch), scratch.numel(), st)

    t_gtq = time_kernel(gtq)
    t_gx = time_kernel(gx)
    flop = 2.0 * rows * cfg.n * cfg.k
    dom_name, dom_t, dom_k = ("gemm_gtq (B = Q^T G, DMMA)", t_gtq, "k_gtq") if t_gtq >= t_gx \
        else ("gemm_gx (Y = G X, DMMA)", t_gx, "k_gx")
    achieved = flop / dom_t / 1e12
    # sketch-GEMM TFLOP/s over the 2q+2 G passes of both matrices (per rank),
    # from the per-launch times scaled by each matrix's rows
    per = cfg.q + 1
    gemm_time = per * (t_gtq + t_gx) * (cfg.m + cfg.p) / cfg.m
    sketch = cfg.flops / world / gemm_time / 1e12
    del Q, Bo, Xt, Y, scratch
    roof = {"bound": "tensor", "kernel": dom_name, "achieved": achieved,
            "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_DMMA_PEAK_TFLOPS,
            "traffic": committed_traffic(cfg.name, dom_k) if world == 1 else None,
            "flop_per_launch": flop, "launch_us": dom_t * 1e6,
            "peak_source": "measured FP64 DMMA issue peak (tools/fp64_peak.cu, "
                           "profiles/r01_fp64_peak.log; MEASURED_PEAKS.json has no FP64 figure)",
            "share_of_step": per * 2 * dom_t * (cfg.m + cfg.p) / cfg.m / steps_time_per_pair}
    return roof, sketch, {"gemm_gtq": t_gtq * 1e6, "gemm_gx": t_gx * 1e6}


def run_ours_sharded(args, rank, world):
    """ONE pair per step, G1/G2 row-sharded over the ranks (genes): each
    matrix chain is one native rgsv_sketch_project_sharded call per rank with
    every ||G||^2, k x k Gram, Z^T and B partial all-reduced in-stream by NCCL
    communicators owned by librgsv (dist.Comm), the two chains on two
    streams, the small GSVD on rank 0 and broadcast; the whole pair is one
    CUDA graph per rank after warm-up. Strong scaling. fp32 configs (cfg4)
    take the tf32x3 tensor-core chain with the same reductions."""
    import torch
    import torch.distributed as dist

    from paper_2404_09459_b200 import _native
    from paper_2404_09459_b200 import device as dv
    from paper_2404_09459_b200 import dist as rdist
    from paper_2404_09459_b200.workloads import CONFIGS, make_pair

    cfg = CONFIGS[args.config]
    f32 = cfg.dtype == "f32"
    dt = torch.float32 if f32 else torch.float64
    gen = torch.Generator(device="cuda").manual_seed(77)  # B shared by all ranks
    b1 = torch.randn((cfg.n, cfg.s), generator=gen, device="cuda", dtype=dt)
    b2 = torch.cat([b1[:, : cfg.shared],
                    torch.randn((cfg.n, cfg.s - cfg.shared), generator=gen, device="cuda",
                                dtype=dt)], dim=1)
    d = (10.0 ** (-cfg.decay * torch.arange(cfg.s, device="cuda", dtype=torch.float64)
                  / cfg.s)).to(dt)
    r0, r1 = rdist.shard_rows(cfg.m, rank, world)
    s0, s1 = rdist.shard_rows(cfg.p, rank, world)
    g1 = device_matrix(r1 - r0, cfg, 1000 + rank, b1, d, dt)
    g2 = device_matrix(s1 - s0, cfg, 2000 + rank, b2, d, dt)
    comm = rdist.default_comm()

    def step(a, b, i):
        return rdist.compute_gsv_sharded(a, b, cfg.m, cfg.p, cfg.n, cfg.k, cfg.q, seed=i,
                                         comm=comm)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        step(g1, g2, i)
    barrier()
    clocks = Clocks(torch.cuda.current_device()) if rank == 0 else None
    l0 = _native.lib().rgsv_launch_count() + dv.GRAPH_REPLAYS[1]
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        res = step(g1, g2, i)
    e1.record(stream)
    barrier()
    launches = _native.lib().rgsv_launch_count() + dv.GRAPH_REPLAYS[1] - l0
    clk = clocks.stop() if clocks else None
    tt = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max = float(tt.item())
    value = args.steps / t_max

    # e2e: every step copies this rank's shards from pinned host memory
    h1 = g1.cpu().pin_memory()
    h2 = g2.cpu().pin_memory()
    d1 = torch.empty_like(g1)
    d2 = torch.empty_like(g2)

    def e2e_step(i):
        d1.copy_(h1, non_blocking=True)
        d2.copy_(h2, non_blocking=True)
        return step(d1, d2, i)

    for i in range(min(2, max(args.warmup, 2))):
        e2e_step(i)
    barrier()
    ne = max(3, args.steps // 2)
    e0.record(stream)
    for i in range(ne):
        e2e_step(i)
    e1.record(stream)
    barrier()
    te = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = ne / float(te.item())
    h2d = (h1.numel() + h2.numel()) * h1.element_size()
    d2h = int(res.report.plan.pk.nbytes) if hasattr(res.report, "plan") and res.report.plan \
        else (6 * cfg.n + 8) * 8
    del d1, d2, h1, h2

    if f32:
        roof, sketch, kus = None, None, None
    else:
        roof, sketch, kus = fp64_gemm_roofline(cfg, dv.to_device(g1, "g1"), r1 - r0,
                                               t_max / args.steps, world)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not f32:
        hg1, hg2 = make_pair(cfg)
        cpu = cpu_baseline(cfg, args.cpu_sample_seconds, hg1, hg2)
        del hg1, hg2
    if rank == 0:
        peak = MEASURED_BF16_TFLOPS / 6.0 if f32 else FP64_DMMA_PEAK_TFLOPS
        eff = cfg.flops * value / world / 1e12
        line = {
            "metric": metric(cfg),
            "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 (3xTF32 tensor cores)" if f32 else "f64",
            "data": "synthetic (device-generated per rank with the workloads.py recipe)",
            "config": {"workload": workload_desc(cfg), "g_bytes": cfg.g_bytes,
                       "step": "one pair per step, row-sharded over the ranks",
                       "parallelism": f"row-sharded x{world} ({comm.mode}: all-reduce of "
                                      "||G||^2 / Gram / Z / B partials, rank-0 small GSVD "
                                      "broadcast)",
                       "l2": "inputs larger than L2"},
            "roofline": roof or {"bound": "tensor", "kernel": "whole chain (GEMM flops / step)",
                                 "achieved": eff, "peak": peak, "unit": "TFLOP/s",
                                 "frac": eff / peak, "traffic": None,
                                 "peak_source": "3xTF32 = measured bf16 / 6"},
            "sketch_gemm_tflops_per_gpu": sketch,
            "sketch_gemm_frac_of_peak": sketch / FP64_DMMA_PEAK_TFLOPS if sketch else None,
            "chain_tflops_per_gpu": eff,
            "kernel_us": kus,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "path": "dist.compute_gsv_sharded() with each rank's shards copied H2D "
                            "from pinned host memory every step and the report read back"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "check": {"r": int(res.r), "s": int(res.s)},
        }
        print(json.dumps(line), flush=True)


def run_ours(args, rank, world):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2404_09459_b200 as rg
    from paper_2404_09459_b200 import _native
    from paper_2404_09459_b200 import device as dv
    from paper_2404_09459_b200.engine import run_device_pipeline
    from paper_2404_09459_b200.workloads import CONFIGS, make_pair

    cfg = CONFIGS[args.config]
    # concurrent pairs per step: 64 for the tiny cfg0 pairs, 8 for cfg1,
    # two genome-scale cfg2 pairs (2 x 11.2 GB)
    # (cfg0: 6483 / 7114 / 7863 pairs/s at 8 / 32 / 64 concurrent pairs;
    #  cfg2: 14.14 / 14.66 / 14.71 pairs/s and e2e 4.18 / 4.53 / 4.69 at 1 / 2 / 3)
    B = max(1, args.batch or (64 if cfg.g_bytes * 64 <= 1e9 else
                              8 if cfg.g_bytes * 8 <= 24e9 else
                              2 if cfg.g_bytes * 2 <= 24e9 else 1))
    hosts = [make_pair(cfg, data_seed=cfg.data_seed + rank * B + b) for b in range(B)]
    pairs = [rg.GmpPair.resident(torch.from_numpy(h1).cuda(), torch.from_numpy(h2).cuda())
             for h1, h2 in hosts]
    pair = pairs[0]
    g1h, g2h = hosts[0]

    def opts(seed):
        return rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, seed, cfg.q))

    base = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step(i):
        return rg.compare_batch(pairs, base, seeds=[i * B + b for b in range(B)])

    for i in range(args.warmup):
        step(i)

    # ---- device-resident throughput: B concurrent pairs per step
    barrier()
    clocks = Clocks(torch.cuda.current_device()) if rank == 0 else None
    l0 = _native.lib().rgsv_launch_count() + dv.GRAPH_REPLAYS[1]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    barrier()
    launches = _native.lib().rgsv_launch_count() + dv.GRAPH_REPLAYS[1] - l0
    t = e0.elapsed_time(e1) * 1e-3
    clk = clocks.stop() if clocks else None
    tt = torch.tensor([t], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max = float(tt.item())
    value = args.steps * B * world / t_max
    # kernels per pair: the graph replays what one eager capture launched
    plan = dv.batch_plan(B, cfg.m, cfg.p, cfg.n, cfg.k, cfg.k)

    # ---- single-pair latency (one pair per step, same pipeline)
    for i in range(2):
        run_device_pipeline(pair, opts(i))
    torch.cuda.synchronize()
    e0.record(stream)
    nlat = max(3, args.steps // 2)
    for i in range(nlat):
        run_device_pipeline(pair, opts(i))
    e1.record(stream)
    torch.cuda.synchronize()
    latency_ms = e0.elapsed_time(e1) / nlat

    # ---- end to end through the public API from pinned host memory
    pinned = [(torch.from_numpy(h1).pin_memory(), torch.from_numpy(h2).pin_memory())
              for h1, h2 in hosts]

    def e2e_step(i):
        # host (g1, g2) pairs: compare_batch streams them in (H2D of pair b+1
        # overlaps the compute of pair b) and reads every report back
        return rg.compare_batch(pinned, base, seeds=[i * B + b for b in range(B)])

    for i in range(min(2, args.warmup)):
        e2e_step(i)
    barrier()
    e0.record(stream)
    for i in range(args.steps):
        reps = e2e_step(i)
    e1.record(stream)
    barrier()
    rep = reps[0]
    te = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = args.steps * B * world / float(te.item())
    sub = plan.plans[0]
    h2d = B * (g1h.nbytes + g2h.nbytes + 16)
    d2h = B * sub.pk.nbytes

    # ---- dominant kernel, timed live (CUDA events on its stream)
    step_s = t_max / (args.steps * B)
    roof, sketch_tflops, kus = fp64_gemm_roofline(cfg, pair.g1, cfg.m, step_s)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # N=1 only (contract)
        cpu = cpu_baseline(cfg, args.cpu_sample_seconds, g1h, g2h)

    if rank == 0:
        line = {
            "metric": metric(cfg),
            "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
            "latency_ms_per_pair": latency_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_desc(cfg),
                       "g_bytes": cfg.g_bytes,
                       "batch": B,
                       "step": f"{B} independent pairs per step, processed concurrently "
                               "(compare_batch, one CUDA graph); Omega seeds step*B + b",
                       "l2": "inputs larger than L2 (%d x G1+G2 = %.0f MB > 126 MB)"
                             % (B, B * cfg.g_bytes / 1e6),
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
            "roofline": roof,
            "sketch_gemm_tflops": sketch_tflops,
            "sketch_gemm_frac_of_peak": sketch_tflops / FP64_DMMA_PEAK_TFLOPS,
            "kernel_us": kus,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "path": "paper_2404_09459_b200.compare_batch() on (g1, g2) pinned host "
                            "arrays: every step streams all pairs H2D (copy stream, each "
                            "pair's compute starts when its own copy lands) and reads every "
                            "report D2H"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "check": {"r": int(rep.spectrum.r), "s": int(rep.spectrum.s), "d1": rep.d1,
                      "d2": rep.d2},
        }
        print(json.dumps(line), flush=True)


def select_mode(args, world: int) -> str:
    """Which timed path a run takes: cfg3's many small pairs are independent
    (replicas at any N); single-pair configs at N > 1 run ONE pair
    row-sharded over the ranks (strong scaling) unless --replicas."""
    from paper_2404_09459_b200.workloads import CONFIGS

    cfg = CONFIGS[args.config]
    if cfg.batch > 1:
        return "batch"
    if args.sharded or (world > 1 and not args.replicas):
        return "sharded"
    return "f32" if cfg.dtype == "f32" else "pairs"


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        # every host core for the CPU reference: torchrun exports
        # OMP_NUM_THREADS=1, under which a threaded OpenBLAS runs its whole
        # thread team on one OpenMP thread (slower than one thread); set it
        # before numpy / OpenBLAS load
        ncpu = str(os.cpu_count() or 1)
        os.environ["OMP_NUM_THREADS"] = ncpu
        os.environ["OPENBLAS_NUM_THREADS"] = ncpu
        run_reference(args, rank, world)
        return
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2404_09459_b200.workloads import CONFIGS

    {"batch": run_ours_batch, "sharded": run_ours_sharded, "f32": run_ours_f32,
     "pairs": run_ours}[select_mode(args, world)](args, rank, world)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
