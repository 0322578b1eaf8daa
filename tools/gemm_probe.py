"""Launch one config's G-pass GEMM shapes a few times (for ncu captures).

    python tools/gemm_probe.py [reps] [cfg1|cfg2]

k_gtq = B = Q^T G (projection / power step), k_gx = Y = G X (sketch / power
step) on G1's shape (m x n) at kp = ceil16(k) columns.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "cfg1"]
m, n, k = cfg.m, cfg.n, cfg.k
kp, ldb = dv.ceil16(k), dv.ceil16(n)
L = _native.lib()
st = dv.sp(torch.cuda.current_stream())
G = torch.randn(m, n, dtype=torch.float64, device="cuda")
Q = torch.randn(m, kp, dtype=torch.float64, device="cuda")
Q[:, k:] = 0
Bo = torch.zeros(kp, ldb, dtype=torch.float64, device="cuda")
Xt = torch.zeros(kp, ldb, dtype=torch.float64, device="cuda")
Xt[:k, :n] = torch.randn(k, n, dtype=torch.float64, device="cuda")
Y = torch.zeros(m, kp, dtype=torch.float64, device="cuda")
S = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
kl = k if k == 120 else kp  # the exact-width tiles the chain uses at k = 120
for _ in range(reps):
    L.rgsv_gemm_gtq(dv.vp(Q), kp, dv.vp(G), n, dv.vp(Bo), ldb, kl, n, m, dv.vp(S), S.numel(), st)
    L.rgsv_gemm_gx(dv.vp(G), n, dv.vp(Xt), ldb, dv.vp(Y), kp, m, kl, n, dv.vp(S), S.numel(), st)
torch.cuda.synchronize()
print("ok", cfg.name, "algorithmic bytes per launch: gtq", 8 * m * n + 8 * m * kp,
      "gx", 8 * m * n + 8 * kp * n)
