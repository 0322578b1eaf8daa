"""Stage times of the cfg4 tf32x3 chain (tf32.tf32_chain), synchronized per
stage, plus the small GSVD."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402
from paper_2404_09459_b200 import tf32 as tf  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS["cfg4"]
frac = float(os.environ.get("FRAC", "1"))
m = int(cfg.m * frac)
n, k, q = cfg.n, cfg.k, cfg.q
g1 = torch.randn((m, n), device="cuda", dtype=torch.float32)
a = dv.DevMatrix(g1, m, n)
T = {}


def t(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    T[label] = T.get(label, 0.0) + (time.perf_counter() - t0) * 1e3
    return out


for rep in range(2):
    T.clear()
    ops = rg.rangefinder._Ops()
    o = tf.TF32Ops()
    kp, ldn = dv.ceil16(k), dv.ceil16(n)
    kq = (kp + 31) // 32 * 32
    glo, ss = t("split G", lambda: o.split_big(a))
    om = t("omega", lambda: dv.omega_device(n, k, [0], ldo=ldn)[0])

    def pass_gx(xt):
        xh, xl = t("split X", lambda: o.split_small(xt, kp, ldn, ldn, rows_out=kq))
        y = torch.empty((m, kq), dtype=torch.float64, device="cuda")
        t("gx", lambda: o.gx(a, glo, xh, xl, y, m, kq, n))
        return y

    def pass_gtq(qm):
        qh, ql = t("split Q", lambda: o.split_small(qm, m, kp, kq))
        out = torch.zeros((kq, ldn), dtype=torch.float64, device="cuda")
        t("gtq", lambda: o.gtq(qh, ql, a, glo, out, kq, n, m))
        return out[:kp]

    y = pass_gx(om)
    qm = t("cholqr mixed (2 pass)", lambda: tf.cholqr_mixed(ops, o, y, m, k, kp, final=q == 0))
    for it in range(q):
        zt = pass_gtq(qm)
        qht = t("cholqr3 wide", lambda: ops.wide_cholqr3(zt.contiguous(), n, ldn, k, kp))
        y = pass_gx(qht)
        qm = t("cholqr mixed (final)",
               lambda: tf.cholqr_mixed(ops, o, y, m, k, kp, final=it == q - 1))
    b = pass_gtq(qm).contiguous()
    t("sumsq B", lambda: ops.sumsq(dv.vp(b), ldn, k, n))
    t("small GSVD + comparative", lambda: dv.small_spectrum(b, k, b, k, n, 1e-10))
    print("rep", rep, " ".join(f"{kk}={v:.1f}ms" for kk, v in T.items()), flush=True)
print("total chain (one matrix, m=%d): %.1f ms" % (m, sum(v for kk, v in T.items() if "small" not in kk)))
