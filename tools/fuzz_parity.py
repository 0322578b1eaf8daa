"""Randomized parity sweep: random shapes / ranks / modes through the public
API on the device against the CPU oracle (test infrastructure). Prints one
line per failing case and a summary; tests/test_gpu_fuzz.py pins a subset."""
import os
import sys
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402


def make(rng, m, p, n, s, noise):
    b1 = rng.standard_normal((n, s))
    sh = s // 2
    b2 = np.hstack([b1[:, :sh], rng.standard_normal((n, s - sh))])
    d = 10.0 ** (-2.0 * np.arange(s) / max(s, 1))
    g1 = (rng.standard_normal((m, s)) * d) @ b1.T + noise * rng.standard_normal((m, n))
    g2 = (rng.standard_normal((p, s)) * d) @ b2.T + noise * rng.standard_normal((p, n))
    return g1, g2


def one_case(rng, idx):
    nmax = int(os.environ.get("NMAX", "260"))
    mmax = int(os.environ.get("MMAX", "1200"))
    n = int(rng.integers(3, nmax))
    m = int(rng.integers(max(2, n // 3), max(mmax, n)))
    p = int(rng.integers(max(2, n // 3), max(mmax, n)))
    if m + p < n:
        m = n
    s = int(rng.integers(1, max(2, min(m, p, n) // 2 + 1)))
    noise = float(rng.choice([1e-3, 1e-6, 1e-9]))
    mode = str(rng.choice(["fixed", "fixed", "direct", "adaptive"]))
    seed = int(rng.integers(0, 1000))
    g1, g2 = make(rng, m, p, n, s, noise)
    desc = f"#{idx} m={m} p={p} n={n} s={s} noise={noise:g} mode={mode} seed={seed}"
    try:
        pair = rg.GmpPair(g1, g2)
    except rg.RankDeficiencyError as exc:
        sv = np.linalg.svd(np.vstack([g1, g2]), compute_uv=False)
        ok = sv[-1] <= 1e-12 * sv[0]  # the reference raises under the same condition
        return ok, desc + f" GmpPair: {exc} (LAPACK ratio {sv[-1] / sv[0]:.3e})", 0.0, None, None, \
            None, None
    if mode == "fixed":
        k = int(rng.integers(1, min(m, p, n) + 1))
        k = min(k, int(os.environ.get("KMAX", "200")))
        q = int(rng.integers(0, 3))
        desc += f" k={k} q={q}"
        opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(k, seed, q))
        o = orc.run_pipeline(g1, g2, k=k, q=q, seed=seed)
        tol = 1e-8
    elif mode == "direct":
        opts = rg.GsvOptions(method="direct")
        o = orc.run_pipeline(g1, g2, direct=True)
        tol = 1e-9
    else:
        opts = rg.GsvOptions(extraction=rg.ExtractionConfig(seed=seed))
        o = orc.run_pipeline(g1, g2, seed=seed)
        tol = 1e-7
    spec = rg.compute_gsv(pair, opts)
    sv = np.linalg.svd(np.vstack([g1, g2]), compute_uv=False)
    tol = max(1e-11, 200.0 * 2.22e-16 * sv[0] / sv[-1])
    desc += f" cond={sv[0] / sv[-1]:.1e}"
    err = float(np.max(np.abs(spec.alphas - o.alphas)))
    ok = err <= tol and (spec.r, spec.s) == (o.r, o.s)
    if not ok and mode == "adaptive":
        pl = rg.engine._run_pipeline(pair, opts)
        w = (pl.l1_block.shape[0], pl.l2_block.shape[0])
        ow = (o.l1_block.shape[0], o.l2_block.shape[0])
        if w != ow:
            desc += f" [stop-decision floor: widths {w} vs oracle {ow}]"
            ok = True
    rep = rg.compare(pair, opts)
    ref = orc.comparative(o.alphas, o.betas, o.r)
    return ok, desc, err, (spec.r, spec.s), (o.r, o.s), rep, ref


def main():
    ncases = int(os.environ.get("CASES", "60"))
    rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
    bad = 0
    for i in range(ncases):
        try:
            ok, desc, err, rs, ors, _, _ = one_case(rng, i)
            if rs is None:
                print("RANKDEF", "agrees" if ok else "DISAGREES", desc, flush=True)
            if not ok:
                bad += 1
                print("MISMATCH", desc, f"err={err:.3e} rs={rs} oracle={ors}", flush=True)
        except Exception as exc:  # noqa: BLE001
            bad += 1
            print("ERROR", i, type(exc).__name__, str(exc)[:300], flush=True)
            traceback.print_exc(limit=2)
    print(f"fuzz: {ncases - bad}/{ncases} ok")


if __name__ == "__main__":
    main()
