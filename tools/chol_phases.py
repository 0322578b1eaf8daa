"""Per-block phase split (clock64) of the one-CTA blocked Cholesky k_chol_blk
at kp = 128: diagonal 8x8 factor (thread 0), panel / block-row tiles, DMMA
rank-8 updates."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402

L = _native.lib()
st = dv.sp(torch.cuda.current_stream())
k = kp = 128
x = np.random.default_rng(1).standard_normal((3 * k, k))
G = torch.from_numpy(x.T @ x).cuda()
linv = torch.zeros(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
status = torch.zeros(1, dtype=torch.int32, device="cuda")
prof = torch.zeros(128, dtype=torch.int64, device="cuda")
for _ in range(3):
    L.rgsv_debug_chol_profile(dv.vp(G), k, kp, dv.vp(linv), dv.vp(prof), dv.vp(status), st)
torch.cuda.synchronize()
p = prof.cpu().numpy()
tot = [0, 0, 0]
for jb in range(16):
    b = 1 + 4 * jb
    d = [p[b + 1] - p[b], p[b + 2] - p[b + 1], p[b + 3] - p[b + 2]]
    for i in range(3):
        tot[i] += d[i]
    if jb < 3 or jb > 13:
        print(f"block {jb:2d}: diag {d[0]:6d}  panel {d[1]:6d}  update {d[2]:6d} cycles")
print("total cycles: diag %d  panel %d  update %d  (all %d)" % (tot[0], tot[1], tot[2], p[64] - p[0] if p[64] else sum(tot)))
