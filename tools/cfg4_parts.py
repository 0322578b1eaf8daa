"""cfg4 part timings: tall Gram / TRSM / Cholesky of the fp64 CholeskyQR3,
the small GSVD, and one whole compare() call (synchronized)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS["cfg4"]
m, n, k = cfg.m, cfg.n, cfg.k
kp = dv.ceil16(k)
ops = rg.rangefinder._Ops()


def t(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {(time.perf_counter() - t0) * 1e3 / reps:9.2f} ms", flush=True)


y = torch.randn((m, kp), device="cuda", dtype=torch.float64)
gram = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
q = torch.zeros((m, kp), dtype=torch.float64, device="cuda")
linv = torch.eye(kp, dtype=torch.float64, device="cuda")
t("gram Y^T Y (gemm_gtq, fp64)", lambda: ops.gtq(dv.vp(y), kp, dv.vp(y), kp, dv.vp(gram), kp, kp, kp, m))
t("gram lower (rgsv_gemm_gram_lower, fp64)", lambda: ops.gram(dv.vp(y), kp, kp, m, dv.vp(gram)))
t("trsm Y Linv (gemm_gx, fp64)", lambda: ops.gx(dv.vp(y), kp, dv.vp(linv), kp, dv.vp(q), kp, m, kp, kp))
g = y.T @ y
t("chol_inv (kp=%d)" % kp, lambda: ops.chol(g, k, kp, m))
t("cholqr3 tall", lambda: ops.cholqr3(y, m, k, kp))
del y, q
b1 = torch.randn((kp, dv.ceil16(n)), device="cuda", dtype=torch.float64)
b2 = torch.randn((kp, dv.ceil16(n)), device="cuda", dtype=torch.float64)
t("small GSVD + comparative (l=576)", lambda: dv.small_spectrum(b1, k, b2, k, n, 1e-10))
del b1, b2
g1 = torch.randn((m, n), device="cuda", dtype=torch.float32)
g2 = torch.randn((cfg.p, n), device="cuda", dtype=torch.float32)
pair = rg.GmpPair.resident(g1, g2)
opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(k, 0, cfg.q))
t("compare() whole pair", lambda: rg.compare(pair, opts), reps=2)
a = dv.DevMatrix(g1, m, n)
t("tf32_chain G1", lambda: rg.tf32.tf32_chain(a, k, cfg.q, 0), reps=2)
