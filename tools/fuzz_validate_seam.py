"""Randomized sweep of GmpPair's stacked-rank validation (shapes around the
Householder / CholeskyQR route boundary, graded conditioning, exact
deficiencies) against numpy's verdict, and of engine.spectrum_from_l_blocks
on random L blocks against the oracle. Test infrastructure."""
import os
import sys
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from oracle import rgsv_oracle as orc  # noqa: E402


def validate_case(rng, idx):
    n = int(rng.integers(2, 700))
    rows = int(rng.integers(n, 4000))
    kind = str(rng.choice(["gauss", "graded", "dupcol", "zerocol", "borderline"]))
    s = rng.standard_normal((rows, n))
    if kind == "graded":
        u, _ = np.linalg.qr(s)
        v, _ = np.linalg.qr(rng.standard_normal((n, n)))
        s = (u * np.logspace(0, -float(rng.uniform(2, 11)), n)) @ v.T
    elif kind == "borderline":
        u, _ = np.linalg.qr(s)
        v, _ = np.linalg.qr(rng.standard_normal((n, n)))
        s = (u * np.logspace(0, -float(rng.uniform(11.3, 12.7)), n)) @ v.T
    elif kind == "dupcol" and n > 2:
        s[:, -1] = s[:, 0] + s[:, 1]
    elif kind == "zerocol":
        s[:, int(rng.integers(0, n))] = 0.0
    cut = int(rng.integers(1, rows))
    desc = f"validate #{idx} {kind} rows={rows} n={n} cut={cut}"
    sv = np.linalg.svd(s, compute_uv=False)
    ratio = sv[-1] / sv[0]
    expect_raise = ratio <= 1e-12
    try:
        pair = rg.GmpPair(s[:cut], s[cut:])
        raised = False
    except rg.RankDeficiencyError:
        raised = True
    except rg.ConvergenceError as exc:
        return False, desc + f" ratio={ratio:.2e} ConvergenceError: {exc}"
    desc += f" ratio={ratio:.2e} raised={raised}"
    if 3e-13 < ratio < 3e-12:   # within rounding of the threshold: either verdict is right
        return True, desc
    if raised != expect_raise:
        return False, desc
    if not raised:
        ok = abs(pair.stack_norm2 - sv[0]) <= 1e-11 * sv[0] and \
            abs(1.0 / pair.stack_pinv_norm - sv[-1]) <= max(0.02 * sv[-1], 1e-14 * sv[0])
        return ok, desc + f" smax={pair.stack_norm2:.6e}/{sv[0]:.6e} smin={1 / pair.stack_pinv_norm:.4e}/{sv[-1]:.4e}"
    return True, desc


def seam_case(rng, idx):
    n = int(rng.integers(2, 300))
    l1 = int(rng.integers(1, 400))
    l2 = int(rng.integers(1, 400))
    r = min(l1 + l2, n)
    q, _ = np.linalg.qr(rng.standard_normal((l1 + l2, r)))
    if rng.random() < 0.4 and r > 2:   # force exact zero / one GSVs: zero out part of a block
        z = int(rng.integers(1, r))
        q[:l1, :z] = 0.0
        q, _ = np.linalg.qr(q)
    desc = f"seam #{idx} l1={l1} l2={l2} n={n}"
    try:
        o = orc.spectrum_from_l_blocks(q[:l1], q[l1:], n, 1e-10)
    except Exception as exc:  # noqa: BLE001
        try:
            rg.engine.spectrum_from_l_blocks(q[:l1], q[l1:], n, 1e-10)
        except Exception as exc2:  # noqa: BLE001
            return type(exc2).__name__ != "RuntimeError", desc + f" both raise ({type(exc).__name__}/{type(exc2).__name__})"
        return False, desc + f" oracle raises {type(exc).__name__}: {exc}, device does not"
    try:
        spec = rg.engine.spectrum_from_l_blocks(q[:l1], q[l1:], n, 1e-10)
    except rg.ConvergenceError as exc:
        sv1 = np.linalg.svd(q[:l1], compute_uv=False)
        sv2 = np.linalg.svd(q[l1:], compute_uv=False)
        return False, desc + (f" r={r} ConvergenceError: {exc}; sv(L1) min {sv1.min():.2e} "
                              f"#<1e-14: {(sv1 < 1e-14).sum()}; sv(L2) min {sv2.min():.2e} "
                              f"#<1e-14: {(sv2 < 1e-14).sum()}")
    al, be, rr, ss = o[0], o[1], o[2], o[3]
    err = max(np.max(np.abs(spec.alphas - al)), np.max(np.abs(spec.betas - be)))
    # sqrt(1 - x^2) completion amplifies one-ulp differences near x = 1 to sqrt(eps)
    ok = (spec.r, spec.s) == (rr, ss) and err <= 4e-8
    return ok, desc + f" err={err:.2e} rs={(spec.r, spec.s)} vs {(rr, ss)}"


def main():
    ncases = int(os.environ.get("CASES", "40"))
    rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
    which = os.environ.get("WHICH", "validate,seam").split(",")
    bad = tot = 0
    for name, fn in (("validate", validate_case), ("seam", seam_case)):
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
    print(f"fuzz validate/seam: {tot - bad}/{tot} ok")


if __name__ == "__main__":
    main()
