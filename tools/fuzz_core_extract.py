"""Randomized sweep of extract_basis with random options (tol, blocksize,
max_cols, trim_tol, exact low rank / decaying / Gaussian inputs) against the
oracle's Alg. 1, and of core.reduced_qr / core.svd / pseudoinverse_norm /
frobenius_norm on random tall, square and wide shapes against numpy. Test
infrastructure; prints failures and a summary."""
import os
import sys
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402


def extract_case(rng, idx):
    m = int(rng.integers(2, 3000))
    n = int(rng.integers(2, 400))
    kind = str(rng.choice(["lowrank", "decay", "gauss"]))
    if kind == "lowrank":
        r = int(rng.integers(1, max(2, min(m, n) // 2)))
        g = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    elif kind == "decay":
        r = min(m, n)
        u, _ = np.linalg.qr(rng.standard_normal((m, r)))
        v, _ = np.linalg.qr(rng.standard_normal((n, r)))
        g = (u * 10.0 ** (-6.0 * np.arange(r) / r)) @ v.T
    else:
        g = rng.standard_normal((m, n))
    blocksize = int(rng.choice([1, 3, 8, 17, 50, 100, 128, 200]))
    max_cols = None if rng.random() < 0.5 else int(rng.integers(1, min(m, n) + 1))
    # tolerances well above the sqrt(eps) cancellation floor of the residual estimate
    tol = None if rng.random() < 0.3 else float(np.linalg.norm(g) * 10.0 ** rng.uniform(-6, -1))
    trim_tol = float(rng.choice([1e-12, 1e-8, 0.0]))
    seed = int(rng.integers(0, 1000))
    desc = (f"extract #{idx} {kind} m={m} n={n} bs={blocksize} max_cols={max_cols} "
            f"tol={tol} trim={trim_tol:g} seed={seed}")
    cfg = rg.ExtractionConfig(tol=tol, blocksize=blocksize, seed=seed, max_cols=max_cols,
                              trim_tol=trim_tol)
    res = rg.extract_basis(g, cfg)
    ob = orc.extract_basis(g, tol, blocksize, seed, max_cols, trim_tol, 0)
    msgs = []
    gn = np.linalg.norm(g)
    # default tol = 1e-10 |G| sits below the estimator's sqrt(eps) floor: the
    # final converged flag is the reference's own coin flip there
    if tol is None:
        if kind == "gauss" and (list(res.block_widths) != list(ob.block_widths)
                                or res.iterations != ob.iterations):
            msgs.append(f"loop differs: widths {res.block_widths} vs {ob.block_widths}")
    elif list(res.block_widths) != list(ob.block_widths) or res.converged != ob.converged \
            or res.iterations != ob.iterations:
        msgs.append(f"loop differs: widths {res.block_widths} vs {ob.block_widths}, "
                    f"conv {res.converged}/{ob.converged}")
    elif len(res.residual_history) != len(ob.residual_history) or \
            np.max(np.abs(np.array(res.residual_history) - np.array(ob.residual_history))) \
            > 1e-6 * gn:
        msgs.append(f"history differs {res.residual_history[-3:]} vs {ob.residual_history[-3:]}")
    if kind == "lowrank" and trim_tol == 0.0:
        # columns kept past the rank are orthonormalised rounding noise in both
        # implementations (tools/extract_diag.py): no invariant to check
        return not msgs, desc + " " + "; ".join(msgs)
    q = res.q
    k = q.shape[1]
    if k and np.linalg.norm(q.T @ q - np.eye(k)) > 1e-10 * np.sqrt(k):
        msgs.append(f"orthonormality {np.linalg.norm(q.T @ q - np.eye(k)):.2e}")
    true_res = np.linalg.norm(g - q @ (q.T @ g)) if k else gn
    if abs(true_res - res.residual_history[-1]) > 2e-7 * gn:
        msgs.append(f"residual estimate {res.residual_history[-1]:.3e} vs true {true_res:.3e}")
    return not msgs, desc + " " + "; ".join(msgs)


def core_case(rng, idx):
    rows = int(rng.integers(1, 2500))
    cols = int(rng.integers(1, 300))
    if rng.random() < 0.3:
        rows, cols = cols, rows
    a = rng.standard_normal((rows, cols))
    desc = f"core #{idx} {rows}x{cols}"
    msgs = []
    k = min(rows, cols)
    qf = rg.reduced_qr(a)
    q_ref, r_ref = orc.reduced_qr(a)
    if qf.q.shape != q_ref.shape or qf.r.shape != r_ref.shape:
        msgs.append("qr shapes")
    else:
        if np.linalg.norm(qf.q @ qf.r - a) > 1e-12 * np.linalg.norm(a):
            msgs.append("qr residual")
        if np.linalg.norm(qf.q.T @ qf.q - np.eye(k)) > 1e-12 * np.sqrt(k):
            msgs.append("qr orth")
        if np.max(np.abs(qf.r - r_ref)) > 1e-10 * np.abs(r_ref).max():
            msgs.append(f"qr R vs LAPACK {np.max(np.abs(qf.r - r_ref)):.2e}")
    if abs(rg.frobenius_norm(a) - np.linalg.norm(a)) > 1e-14 * np.linalg.norm(a):
        msgs.append("frobenius")
    if min(rows, cols) <= 400:
        sf = rg.svd(a)
        s_ref = np.linalg.svd(a, compute_uv=False)
        if np.max(np.abs(sf.s - s_ref)) > 1e-12 * s_ref[0]:
            msgs.append("svd values")
        if np.linalg.norm((sf.u * sf.s) @ sf.v.T - a) > 1e-11 * np.linalg.norm(a):
            msgs.append("svd reconstruction")
        if rows >= cols:
            pn = rg.pseudoinverse_norm(a)
            if abs(pn - 1.0 / s_ref[-1]) > 1e-9 / s_ref[-1]:
                msgs.append("pinv norm")
    return not msgs, desc + " " + "; ".join(msgs)


def main():
    ncases = int(os.environ.get("CASES", "40"))
    rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
    which = os.environ.get("WHICH", "extract,core").split(",")
    bad = tot = 0
    for name, fn in (("extract", extract_case), ("core", core_case)):
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
                traceback.print_exc(limit=4)
    print(f"fuzz extract/core: {tot - bad}/{tot} ok")


if __name__ == "__main__":
    main()
