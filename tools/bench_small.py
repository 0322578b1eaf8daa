"""Time the small-GSVD stage (rgsv_small_gsvd) alone at each config's shape.

    python tools/bench_small.py            # default dispatch
    RGSV_HH_MIN=100000 RGSV_BJ_MIN=100000 python tools/bench_small.py   # one-CTA kernels

Also times rgsv_dense_qr (k_hhqr) and rgsv_svd_values (k_bjacobi) alone.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402

L = _native.lib()
st = dv.sp(torch.cuda.current_stream())


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


tag = os.environ.get("TAG", "default")
for (k, n) in ((30, 200), (60, 1000), (16, 64), (120, 4000), (288, 8192)):
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
    us = timed(lambda: _native.check(L.rgsv_small_gsvd(*args), "small_gsvd"))
    s = sv1.cpu().numpy()
    print(f"[{tag}] small_gsvd k={k} n={n}: {us:9.1f} us  status={int(ints[2])}"
          f"  sv1 range [{s.min():.17f}, {s.max():.17f}]", flush=True)

for m in (120, 240, 576, 1024):
    a = torch.randn(m, m, dtype=torch.float64, device="cuda")
    q = torch.empty(m, m, dtype=torch.float64, device="cuda")
    nb = int(L.rgsv_dense_qr_workspace_bytes(m, m))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    us = timed(lambda: _native.check(L.rgsv_dense_qr(dv.vp(a), m, m, None, 0, 0, m, dv.vp(q), m,
                                                     None, 0, 0, dv.vp(ws), nb, st), "qr"))
    err = (q.T @ q - torch.eye(m, dtype=torch.float64, device="cuda")).norm().item()
    print(f"[{tag}] dense_qr {m}x{m}: {us:9.1f} us  |QtQ-I|={err:.2e}", flush=True)

for (r, c) in ((60, 120), (120, 240), (288, 576), (1000, 1000)):
    a0 = torch.randn(r, c, dtype=torch.float64, device="cuda")
    qf = torch.linalg.qr(a0.T)[0].T.contiguous() if r <= c else a0  # orthonormal rows
    for name, src in (("orthonormal", qf), ("gaussian", a0)):
        a = src.clone()
        sv = torch.zeros(min(r, c), dtype=torch.float64, device="cuda")
        ints = torch.zeros(4, dtype=torch.int32, device="cuda")
        nb = int(L.rgsv_svd_values_workspace_bytes(r, c))
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")

        def f():
            a.copy_(src)
            _native.check(L.rgsv_svd_values(dv.vp(a), c, r, c, dv.vp(sv), dv.vp(ints[:2]),
                                            dv.vp(ints[2:3]), dv.vp(ws), nb, st), "svd")

        us = timed(f, reps=3)
        print(f"[{tag}] svd_values {r}x{c} {name}: {us:9.1f} us  status={int(ints[2])}",
              flush=True)
