"""Time the 3xTF32 kernels at cfg4 shapes (G1 rows) over the tuning knobs
(rgsv_tf32_config: BK of gx / gtq, rows per split, TMEM flush interval)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402
from paper_2404_09459_b200 import tf32 as tf  # noqa: E402

m = int(os.environ.get("ROWS", "1000000"))
n, kq = 8192, 288
g = torch.randn((m, n), device="cuda", dtype=torch.float32)
a = dv.DevMatrix(g, m, n)
o = tf.TF32Ops()
lo, _ = o.split_big(a)
xh, xl = o.split_small(torch.randn(kq, n, dtype=torch.float64, device="cuda"), kq, n, n)
qh, ql = o.split_small(torch.randn(m, kq, dtype=torch.float64, device="cuda"), m, kq, kq)
y = torch.empty((m, kq), dtype=torch.float64, device="cuda")
z = torch.zeros((kq, n), dtype=torch.float64, device="cuda")
L = _native.lib()
flop = 2.0 * m * n * kq


def tm(fn, reps=3):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


configs = [(32, 32, 8192, 2, pf) for pf in (0, 2, 4, 8, 16)]
if os.environ.get("FULL_SWEEP"):
    configs = [(16, 16, 8192, 1, 0), (32, 16, 8192, 1, 0), (16, 32, 8192, 1, 0),
               (16, 16, 8192, 2, 0), (32, 32, 8192, 1, 0), (32, 32, 8192, 2, 0)] + configs
for bk, bq, rps, fl, pf in configs:
    os.environ["RGSV_TF32_PREFETCH"] = str(pf)
    L.rgsv_tf32_config(bk, bq, rps, fl)
    tgx = tm(lambda: o.gx(a, lo, xh, xl, y, m, kq, n))
    tgq = tm(lambda: o.gtq(qh, ql, a, lo, z, kq, n, m))
    print(f"bk_gx={bk} bk_gtq={bq} rows/split={rps} flush={fl} l2_prefetch={pf}: gx "
          f"{tgx*1e3:.2f} ms ({flop/tgx/1e12:.1f} TF/s)  gtq {tgq*1e3:.2f} ms "
          f"({flop/tgq/1e12:.1f} TF/s)", flush=True)
