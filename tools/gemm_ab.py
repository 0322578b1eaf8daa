"""A/B timing of the cfg1 GEMM shapes (set RGSV_GEMM_VARIANT before import)."""
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
S = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
ref_b = None


def run(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def gtq():
    L.rgsv_gemm_gtq(dv.vp(Q), kp, dv.vp(G), n, dv.vp(Bo), ldb, kp, n, m, dv.vp(S), S.numel(), st)


def gx():
    L.rgsv_gemm_gx(dv.vp(G), n, dv.vp(Xt), ldb, dv.vp(Y), kp, m, kp, n, dv.vp(S), S.numel(), st)


tq, tx = run(gtq), run(gx)
fl = 2 * m * n * k
ref = (Q[:, :k].T @ G)
err = (Bo[:k, :n] - ref).norm() / ref.norm()
print(f"variant={os.environ.get('RGSV_GEMM_VARIANT', '0')} gtq {tq:.1f} us {fl / tq / 1e6:.2f} TF | "
      f"gx {tx:.1f} us {fl / tx / 1e6:.2f} TF | gtq rel err {err:.2e}")
