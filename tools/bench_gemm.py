"""Time the two GEMM kernels on the configs' shapes (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402

L = _native.lib()
st = dv.sp(torch.cuda.current_stream())
S = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def tm(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


for name, m, n, k in (("cfg1 G1", 20000, 1000, 60), ("cfg1 G2", 16000, 1000, 60),
                      ("cfg0 G1", 2000, 200, 30), ("cfg2 G1", 200000, 4000, 120),
                      ("cfg3 G1", 4000, 64, 16)):
    kp = (k + 15) // 16 * 16
    ldb = (n + 15) // 16 * 16
    G = torch.randn(m, n, dtype=torch.float64, device="cuda")
    Q = torch.randn(m, kp, dtype=torch.float64, device="cuda")
    Bo = torch.zeros(kp, ldb, dtype=torch.float64, device="cuda")
    Xt = torch.randn(kp, ldb, dtype=torch.float64, device="cuda")
    Y = torch.zeros(m, kp, dtype=torch.float64, device="cuda")
    t1 = tm(lambda: L.rgsv_gemm_gtq(dv.vp(Q), kp, dv.vp(G), n, dv.vp(Bo), ldb, kp, n, m,
                                    dv.vp(S), S.numel(), st))
    t2 = tm(lambda: L.rgsv_gemm_gx(dv.vp(G), n, dv.vp(Xt), ldb, dv.vp(Y), kp, m, kp, n,
                                   dv.vp(S), S.numel(), st))
    f = 2.0 * m * n * k
    print(f"{name:8s} gtq {t1*1e6:8.1f} us {f/t1/1e12:6.2f} TF | gx {t2*1e6:8.1f} us "
          f"{f/t2/1e12:6.2f} TF  (algorithmic k={k}, kp={kp})")
    del G, Q, Bo, Xt, Y
