"""Randomized sweep of the batch API (compare_batch on random small shapes:
every k_batch_chain instantiation, ragged sizes) and of recover_gsvd (random
shapes incl. synth_gmp pairs with zero blocks) against the oracle /
reconstruction invariants. Test infrastructure; prints failures + summary."""
import os
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402
from tools.fuzz_parity import make  # noqa: E402


def batch_case(rng, idx):
    k = int(rng.integers(2, 33))
    if rng.random() < 0.6:   # 2k >= n: data-dependent spectrum (s > 0)
        n = int(rng.integers(max(4, k), 2 * k + 1))
    else:                    # 2k < n: the closed-form degenerate spectrum
        n = int(rng.integers(2 * k + 1, 131))
    q = int(rng.integers(0, 3))
    m = int(rng.integers(max(k, n // 2), 5000))
    p = int(rng.integers(max(k, n // 2), 5000))
    if m + p < n:
        m = n
    B = int(rng.integers(1, 7))
    s = int(rng.integers(1, max(2, min(m, p, n) // 2 + 1)))
    noise = float(rng.choice([1e-3, 1e-6, 1e-8]))
    desc = f"batch #{idx} B={B} m={m} p={p} n={n} k={k} q={q} s={s} noise={noise:g}"
    hosts = [make(rng, m, p, n, s, noise) for _ in range(B)]
    seeds = [int(x) for x in rng.integers(0, 10000, B)]
    pairs = [rg.GmpPair.resident(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
             for a, b in hosts]
    opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(k, 0, q))
    reps = rg.compare_batch(pairs, opts, seeds)
    runs = rg.engine.run_device_batch(pairs, opts, seeds)
    worst = 0.0
    for j, (g1, g2) in enumerate(hosts):
        o = orc.run_pipeline(g1, g2, k=k, q=q, seed=seeds[j])
        sv = np.linalg.svd(np.vstack([g1, g2]), compute_uv=False)
        tol = max(1e-11, 200.0 * 2.22e-16 * sv[0] / sv[-1])
        sp = reps[j].spectrum
        err = float(np.max(np.abs(sp.alphas - o.alphas)))
        worst = max(worst, err / tol)
        if (sp.r, sp.s) != (o.r, o.s) or err > tol:
            return False, desc + f" pair {j}: err={err:.2e} tol={tol:.2e} rs={(sp.r, sp.s)} vs {(o.r, o.s)}"
        for basis, ob in ((runs[j].basis1, o.basis1), (runs[j].basis2, o.basis2)):
            h, ho = basis.residual_history, ob.residual_history
            e, eo = h[0] ** 2 - h[1] ** 2, ho[0] ** 2 - ho[1] ** 2
            if abs(h[0] - ho[0]) > 1e-13 * ho[0] or abs(e - eo) > 1e-11 * eo:
                return False, desc + f" pair {j}: energy {e:.17g} vs oracle {eo:.17g}"
        ref = orc.comparative(o.alphas, o.betas, o.r)
        th = ref[1] if isinstance(ref, tuple) else ref["theta"]
        if np.max(np.abs(reps[j].theta - th)) > 10 * tol:
            return False, desc + f" pair {j}: theta differs"
    return True, desc + f" worst err/tol={worst:.2e}"


def recover_case(rng, idx):
    kind = str(rng.choice(["gauss", "synth"]))
    n = int(rng.integers(3, 200))
    method = str(rng.choice(["direct", "randomized"]))
    if kind == "gauss":
        m = int(rng.integers(n, 1500))
        p = int(rng.integers(n, 1500))
        g1 = rng.standard_normal((m, n))
        g2 = rng.standard_normal((p, n))
        pair = rg.GmpPair(g1, g2)
        desc = f"recover #{idx} gauss m={m} p={p} n={n} {method}"
    else:
        m = int(rng.integers(n, 1200))
        p = int(rng.integers(n, 1200))
        frac = float(rng.uniform(0.55, 1.0))
        res = rg.synth_gmp(rg.SynthSpec(m=m, p=p, n=n, rank_frac=frac,
                                        seed=int(rng.integers(0, 999)), field="real"))
        pair = res.pair
        g1, g2 = pair.g1.t.cpu().numpy(), pair.g2.t.cpu().numpy()
        desc = f"recover #{idx} synth m={m} p={p} n={n} frac={frac:.2f} {method} cond={res.condition_r:.1e}"
    opts = rg.GsvOptions(method=method, extraction=rg.ExtractionConfig(tol=1e-12, seed=idx))
    fac = rg.recover_gsvd(pair, opts)
    a, b = fac.spectrum.alphas, fac.spectrum.betas
    e1 = np.linalg.norm(fac.u @ (a[:, None] * fac.r_factor) - g1) / np.linalg.norm(g1)
    e2 = np.linalg.norm(fac.v @ (b[:, None] * fac.r_factor) - g2) / np.linalg.norm(g2)
    ou = np.linalg.norm(fac.u.T @ fac.u - np.eye(n))
    ov = np.linalg.norm(fac.v.T @ fac.v - np.eye(n))
    ok = max(e1, e2) <= 1e-8 and max(ou, ov) <= 1e-8 * np.sqrt(n)
    return ok, desc + f" recon={max(e1, e2):.1e} orth={max(ou, ov):.1e}"


def main():
    ncases = int(os.environ.get("CASES", "40"))
    rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
    which = os.environ.get("WHICH", "batch,recover").split(",")
    bad = tot = 0
    for name, fn in (("batch", batch_case), ("recover", recover_case)):
        if name not in which:
            continue
        for i in range(ncases):
            tot += 1
            try:
                ok, desc = fn(rng, i)
                if not ok:
                    bad += 1
                    print("FAIL", desc, flush=True)
                elif os.environ.get("VERBOSE"):
                    print("ok", desc, flush=True)
            except Exception as exc:  # noqa: BLE001
                bad += 1
                print("ERROR", name, i, type(exc).__name__, str(exc)[:300], flush=True)
                traceback.print_exc(limit=3)
    print(f"fuzz batch/recover: {tot - bad}/{tot} ok")


if __name__ == "__main__":
    main()
