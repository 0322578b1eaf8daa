"""Time rgsv_chol_inv on a near-identity Gram (third-pass fast path) vs a
general SPD Gram, both unshifted."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402

L = _native.lib()
st = dv.sp(torch.cuda.current_stream())
for k in (30, 60):
    kp = (k + 15) // 16 * 16
    rng = np.random.default_rng(k)
    x = rng.standard_normal((k, k))
    for label, a in (("near-I", np.eye(k) + 3e-8 * (x + x.T)), ("general", x @ x.T + k * np.eye(k))):
        G = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
        G[:k, :k] = torch.from_numpy(a)
        linv = torch.zeros(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        args = (dv.vp(G), k, kp, 0, dv.vp(linv), None, None, dv.vp(status), st)
        for _ in range(5):
            L.rgsv_chol_inv(*args)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            L.rgsv_chol_inv(*args)
        e1.record()
        e1.synchronize()
        li = linv[: kp * kp].view(kp, kp).cpu().numpy()[:k, :k]
        err = np.abs(li - np.linalg.inv(np.linalg.cholesky(a))).max()
        print(f"k={k} {label:8s}: {e0.elapsed_time(e1) / 200 * 1e3:7.2f} us  err {err:.1e}")
