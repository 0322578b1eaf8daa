"""Time rgsv_f32_split (lo part + ||G||^2) at cfg4's G1 shape (HBM-bound:
reads G, writes lo) and check ||G||^2 against a chunked fp64 sum."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09459_b200 import device as dv  # noqa: E402
from paper_2404_09459_b200 import tf32 as tf  # noqa: E402

m, n = 1000000, 8192
g = torch.randn((m, n), device="cuda", dtype=torch.float32)
a = dv.DevMatrix(g, m, n)
o = tf.TF32Ops()
lo, ss = o.split_big(a)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    o.split_big(a, lo)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 5
ref = sum(float((g[r:r + 65536].double() ** 2).sum()) for r in range(0, m, 65536))
print(f"split: {t:.2f} ms, {2 * m * n * 4 / t / 1e6:.0f} GB/s; "
      f"||G||^2 rel err {abs(float(ss.item()) - ref) / ref:.2e}")

# small-operand split of a tall fp64 Q (m x 288)
q = torch.randn((m, 288), device="cuda", dtype=torch.float64)
del g, lo
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    qh, ql = o.split_small(q, m, 288, 288)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 5
print(f"split_small (m x 288 fp64 -> hi/lo fp32): {t:.2f} ms, {m * 288 * 16 / t / 1e6:.0f} GB/s")
hv = qh.double() + ql.double()
print(f"hi + lo vs x: max rel {float(((hv - q).abs() / q.abs().clamp_min(1e-300)).max()):.2e}")
