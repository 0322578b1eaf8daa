"""Small L blocks (< 64 vectors: the one-CTA Jacobi) and small batched pairs
with exactly zero / one GSVs against the oracle (exploration)."""
import os
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
bad = tot = 0
for idx in range(60):
    tot += 1
    n = int(rng.integers(2, 60))
    l1 = int(rng.integers(1, 64))
    l2 = int(rng.integers(1, 64))
    r = min(l1 + l2, n)
    q, _ = np.linalg.qr(rng.standard_normal((l1 + l2, r)))
    if rng.random() < 0.6 and r > 2:
        q[:l1, : int(rng.integers(1, r))] = 0.0
        q, _ = np.linalg.qr(q)
    try:
        try:
            o = orc.spectrum_from_l_blocks(q[:l1], q[l1:], n, 1e-10)
        except Exception:  # noqa: BLE001
            continue
        spec = rg.engine.spectrum_from_l_blocks(q[:l1], q[l1:], n, 1e-10)
        err = max(np.max(np.abs(spec.alphas - o[0])), np.max(np.abs(spec.betas - o[1])))
        if (spec.r, spec.s) != (o[2], o[3]) or err > 4e-8:
            bad += 1
            print(f"FAIL seam l1={l1} l2={l2} n={n} err={err:.2e} rs={(spec.r, spec.s)} vs {(o[2], o[3])}")
    except Exception as exc:  # noqa: BLE001
        bad += 1
        print(f"ERROR seam l1={l1} l2={l2} n={n}", type(exc).__name__, str(exc)[:200])
# batched small pairs with zero blocks (synth-like), direct-free: fixed rank k = n (full width)
for idx in range(20):
    tot += 1
    n = int(rng.integers(6, 33))
    k = n // 2 + int(rng.integers(0, n - n // 2 + 1))
    m = int(rng.integers(n + 5, 900))
    p = int(rng.integers(n + 5, 900))
    B = int(rng.integers(1, 5))
    hosts = []
    for _ in range(B):
        res = rg.synth_gmp(rg.SynthSpec(m=m, p=p, n=n, rank_frac=float(rng.uniform(0.6, 1.0)),
                                        seed=int(rng.integers(0, 999)), field="real"))
        hosts.append((res.pair.g1.t.cpu().numpy().copy(), res.pair.g2.t.cpu().numpy().copy()))
    seeds = [int(x) for x in rng.integers(0, 1000, B)]
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(k, 0, 1))
    try:
        pairs = [rg.GmpPair.resident(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
                 for a, b in hosts]
        reps = rg.compare_batch(pairs, opts, seeds)
        for j, (a, b) in enumerate(hosts):
            o = orc.run_pipeline(a, b, k=k, q=1, seed=seeds[j])
            sp = reps[j].spectrum
            err = float(np.max(np.abs(sp.alphas - o.alphas)))
            if (sp.r, sp.s) != (o.r, o.s) or err > 1e-6:
                bad += 1
                print(f"FAIL batch n={n} k={k} m={m} p={p} pair {j}: err={err:.2e} rs={(sp.r, sp.s)} vs {(o.r, o.s)}")
                break
    except Exception as exc:  # noqa: BLE001
        bad += 1
        print(f"ERROR batch n={n} k={k} m={m} p={p} B={B}", type(exc).__name__, str(exc)[:200])
        traceback.print_exc(limit=3)
print(f"fuzz small/zero: {tot - bad}/{tot} ok")
