"""Time the cfg2 G-pass GEMMs (exact-width k = 120) under the current
RGSV_* tuning environment: python tools/gemm_variants.py [reps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
m, n, k, kp = 200000, 4000, 120, 128
L = _native.lib()
st = dv.sp(torch.cuda.current_stream())
G = torch.randn(m, n, dtype=torch.float64, device="cuda")
Q = torch.randn(m, kp, dtype=torch.float64, device="cuda")
Q[:, k:] = 0
Bo = torch.zeros(kp, n, dtype=torch.float64, device="cuda")
S = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def gtq():
    _native.check(L.rgsv_gemm_gtq(dv.vp(Q), kp, dv.vp(G), n, dv.vp(Bo), n, k, n, m, dv.vp(S),
                                  S.numel(), st), "gtq")


for _ in range(3):
    gtq()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    gtq()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
ref = Q[:, :k].T @ G
err = ((Bo[:k] - ref).norm() / ref.norm()).item()
print(f"RGSV_GTQ_EXACT={os.environ.get('RGSV_GTQ_EXACT', '0')}: gtq {ms * 1e3:.0f} us "
      f"{2 * m * n * k / ms / 1e9:.1f} TF  rel err {err:.1e}", flush=True)
