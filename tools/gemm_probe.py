"""Launch the cfg1 GEMM shapes a few times (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402

m, n, k = 20000, 1000, 60
kp, ldb = 64, 1008
L = _native.lib()
st = dv.sp(torch.cuda.current_stream())
G = torch.randn(m, n, dtype=torch.float64, device="cuda")
Q = torch.randn(m, kp, dtype=torch.float64, device="cuda")
Bo = torch.zeros(kp, ldb, dtype=torch.float64, device="cuda")
Xt = torch.randn(kp, ldb, dtype=torch.float64, device="cuda")
Y = torch.zeros(m, kp, dtype=torch.float64, device="cuda")
S = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    L.rgsv_gemm_gtq(dv.vp(Q), kp, dv.vp(G), n, dv.vp(Bo), ldb, kp, n, m, dv.vp(S), S.numel(), st)
    L.rgsv_gemm_gx(dv.vp(G), n, dv.vp(Xt), ldb, dv.vp(Y), kp, m, kp, n, dv.vp(S), S.numel(), st)
torch.cuda.synchronize()
print("ok")
