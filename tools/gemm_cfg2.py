"""Time the cfg2 projection GEMM (B = Q^T G, 128 x 4000 over 200000 rows)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402

m, n, kp = 200000, 4000, 128
L = _native.lib()
st = dv.sp(torch.cuda.current_stream())
G = torch.randn(m, n, dtype=torch.float64, device="cuda")
Q = torch.randn(m, kp, dtype=torch.float64, device="cuda")
Bo = torch.zeros(kp, n, dtype=torch.float64, device="cuda")
S = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
f = lambda: L.rgsv_gemm_gtq(dv.vp(Q), kp, dv.vp(G), n, dv.vp(Bo), n, kp, n, m, dv.vp(S), S.numel(), st)
for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
ref = Q[:, :120].T @ G
err = ((Bo[:120] - ref).norm() / ref.norm()).item()
print(f"cfg2 gtq {ms:.2f} ms  {2 * m * n * 120 / ms / 1e9:.1f} TF (k=120)  rel err {err:.1e}")
