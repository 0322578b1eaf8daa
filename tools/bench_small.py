"""Time the small-GSVD stage (rgsv_small_gsvd) alone for cfg-like shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402

L = _native.lib()
st = dv.sp(torch.cuda.current_stream())
for (k, n) in ((30, 200), (60, 1000), (16, 64), (120, 4000)):
    kp = (k + 15) // 16 * 16
    ldb = (n + 15) // 16 * 16
    rng = np.random.default_rng(k)
    b1 = torch.zeros((kp, ldb), dtype=torch.float64, device="cuda")
    b2 = torch.zeros((kp, ldb), dtype=torch.float64, device="cuda")
    b1[:k, :n] = torch.from_numpy(rng.standard_normal((k, n)))
    b2[:k, :n] = torch.from_numpy(rng.standard_normal((k, n)))
    nb = int(L.rgsv_small_gsvd_workspace_bytes(k, k, n))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    sv1 = torch.zeros(k, dtype=torch.float64, device="cuda")
    sv2 = torch.zeros(k, dtype=torch.float64, device="cuda")
    ints = torch.zeros(4, dtype=torch.int32, device="cuda")
    args = (dv.vp(b1), ldb, k, dv.vp(b2), ldb, k, n, dv.vp(sv1), dv.vp(sv2), dv.vp(ints[:2]),
            dv.vp(ints[2:3]), dv.vp(ws), nb, st)
    for _ in range(3):
        L.rgsv_small_gsvd(*args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        L.rgsv_small_gsvd(*args)
    e1.record()
    e1.synchronize()
    s = sv1.cpu().numpy()
    print(f"small_gsvd k={k} n={n}: {e0.elapsed_time(e1) / 20 * 1e3:9.1f} us  status={int(ints[2])}"
          f"  sv1 range [{s.min():.17f}, {s.max():.17f}]")

# phase stamps of one l = 60 Householder (owner phase / apply phase per column)
k, n = 30, 200
b1 = torch.from_numpy(np.random.default_rng(0).standard_normal((k, 208))).cuda()
b2 = torch.from_numpy(np.random.default_rng(1).standard_normal((k, 208))).cuda()
qq = torch.zeros((64, 64), dtype=torch.float64, device="cuda")
prof = torch.zeros(64, dtype=torch.int64, device="cuda")
for _ in range(3):
    L.rgsv_debug_householder_profile(dv.vp(b1), 208, k, dv.vp(b2), 208, k, dv.vp(qq), 64,
                                     dv.vp(prof), st)
torch.cuda.synchronize()
p = prof.cpu().numpy()
for j in range(6):
    print(f"col {j}: owner {p[3*j+1]-p[3*j]} cycles, apply {p[3*j+2]-p[3*j+1]} cycles")
print("factorization total", p[30] - p[0], "dorg2r", p[31] - p[30])
