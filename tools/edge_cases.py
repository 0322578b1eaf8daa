"""Edge cases around rank deficiency, device vs oracle (exploration)."""
import os
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402

rng = np.random.default_rng(0)
low = rng.standard_normal((900, 6)) @ rng.standard_normal((6, 80))
full = rng.standard_normal((700, 80))
noisy = rng.standard_normal((700, 6)) @ rng.standard_normal((6, 80)) + 1e-3 * rng.standard_normal((700, 80))


def attempt(name, fn):
    try:
        print(name, "->", fn(), flush=True)
    except Exception as exc:  # noqa: BLE001
        print(name, "-> EXC", type(exc).__name__, str(exc)[:200], flush=True)
        traceback.print_exc(limit=3)


def eb(q):
    res = rg.extract_basis(low, rg.ExtractionConfig.fixed_rank(20, 3, q))
    ob = orc.fixed_rank_basis(low, 20, q, 3)
    return (res.q.shape, ob.q.shape, f"{np.linalg.norm(low - res.q @ (res.q.T @ low)):.1e}",
            res.residual_history[-1], ob.residual_history[-1])


def gsv(q, g2):
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(20, 3, q))
    spec = rg.compute_gsv(rg.GmpPair(low, g2, check_rank=False), opts)
    o = orc.run_pipeline(low, g2, k=20, q=q, seed=3)
    return (spec.r, spec.s), (o.r, o.s), f"{np.max(np.abs(spec.alphas - o.alphas)):.1e}"


def batch(q):
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(20, 0, q))
    pairs = [rg.GmpPair.resident(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
             for a, b in ((full[:, :48].copy(), noisy[:, :48].copy()),
                          (low[:700, :48].copy(), noisy[:, :48].copy()))]
    reps = rg.compare_batch(pairs, opts, [5, 7])
    out = []
    for j, (a, b) in enumerate(((full[:, :48], noisy[:, :48]), (low[:700, :48], noisy[:, :48]))):
        o = orc.run_pipeline(a, b, k=20, q=q, seed=[5, 7][j])
        sp = reps[j].spectrum
        out.append(((sp.r, sp.s), (o.r, o.s), f"{np.max(np.abs(sp.alphas - o.alphas)):.1e}"))
    return out


def zero_g1():
    z = np.zeros((50, 80))
    opts = rg.GsvOptions()
    spec = rg.compute_gsv(rg.GmpPair(z, rng.standard_normal((200, 80))), opts)
    o = orc.run_pipeline(z, rng.standard_normal((200, 80)))
    return (spec.r, spec.s), (o.r, o.s)


for q in (0, 1, 2):
    attempt(f"extract_basis fixed k=20 q={q} on rank 6", lambda q=q: eb(q))
for q in (0, 1):
    attempt(f"compute_gsv fixed q={q}, g1 rank 6, g2 noisy", lambda q=q: gsv(q, noisy))
    attempt(f"compute_gsv fixed q={q}, g1 rank 6, g2 full", lambda q=q: gsv(q, full))
for q in (0, 1):
    attempt(f"compare_batch q={q} with a rank-deficient pair", lambda q=q: batch(q))
attempt("zero g1, adaptive default", zero_g1)
