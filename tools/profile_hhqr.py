"""Phase timeline of one k_hhqr launch (globaltimer stamps of CTA 0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402

L = _native.lib()
st = dv.sp(torch.cuda.current_stream())
for m in [int(x) for x in (sys.argv[1:] or ["240", "576"])]:
    a = torch.randn(m, m, dtype=torch.float64, device="cuda")
    q = torch.empty(m, m, dtype=torch.float64, device="cuda")
    nb = int(L.rgsv_dense_qr_workspace_bytes(m, m))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    prof = torch.zeros(256, dtype=torch.int64, device="cuda")
    for _ in range(3):
        _native.check(L.rgsv_debug_dense_qr_profile(dv.vp(a), m, m, m, dv.vp(q), dv.vp(ws), nb,
                                                    dv.vp(prof), st), "prof")
    torch.cuda.synchronize()
    p = prof.cpu().numpy()
    n = int(p[255])
    t = (p[:n] - p[0]) / 1e3
    npan = (m + 31) // 32 if m <= 640 else (m + 15) // 16
    print(f"M=N={m}: {n} stamps, total {t[-1]:.1f} us, {npan} panels")
    # layout: [0]=start; per panel: begin, after panel, after barrier, after trailing (if any)
    k = 1
    rows = []
    for pi in range(npan):
        b = t[k]
        ap = t[k + 1]
        ab = t[k + 2]
        k += 3
        tr = None
        if pi < npan - 1:
            tr = t[k]
            k += 1
        rows.append((pi, ap - b, ab - ap, (tr - ab) if tr is not None else 0.0))
    for r in rows[:4] + rows[-2:]:
        print("  panel %2d: factor %7.1f us  barrier %6.1f us  trailing %7.1f us" % r)
    print("  sum factor %.1f  barrier %.1f  trailing %.1f" % tuple(
        sum(r[i] for r in rows) for i in (1, 2, 3)))
    pp = p[128:176]
    if pp[40]:
        b = pp[40]
        print("  panel 0 detail (us): load %.1f, col0 %.1f, cols 1..%d each ~%.2f, writeback %.1f, form_t %.1f" % (
            (pp[0] - b) / 1e3, (pp[2] - pp[1]) / 1e3, 31, (pp[32] - pp[2]) / 30e3,
            (pp[33] - pp[32]) / 1e3, (pp[34] - pp[33]) / 1e3))
    qs = t[k:n]
    print("  Q phase: %.1f us over %d stamps; first steps %s" % (
        qs[-1] - qs[0], len(qs), np.round(np.diff(qs)[:6], 1)))
