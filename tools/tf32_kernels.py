"""Run the 3xTF32 tcgen05 kernels once each at cfg4 column shapes (for ncu):
f32_split, tf32x3_gx (Y = G X^T, N = 288) and tf32x3_gtq (Q^T G, split-K)
on an M-row fp32 G (default 200000 rows x 8192)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_09459_b200 import device as dv  # noqa: E402
from paper_2404_09459_b200 import tf32 as tf  # noqa: E402

m = int(os.environ.get("ROWS", "200000"))
n, kq = 8192, 288
reps = int(os.environ.get("REPS", "1"))
g = torch.randn((m, n), device="cuda", dtype=torch.float32)
a = dv.DevMatrix(g, m, n)
o = tf.TF32Ops()
lo, _ = o.split_big(a)
xh, xl = o.split_small(torch.randn(kq, n, dtype=torch.float64, device="cuda"), kq, n, n)
qh, ql = o.split_small(torch.randn(m, kq, dtype=torch.float64, device="cuda"), m, kq, kq)
y = torch.empty((m, kq), dtype=torch.float64, device="cuda")
z = torch.zeros((kq, n), dtype=torch.float64, device="cuda")
for _ in range(reps):
    o.gx(a, lo, xh, xl, y, m, kq, n)
    o.gtq(qh, ql, a, lo, z, kq, n, m)
torch.cuda.synchronize()
print("ok", float(y[0, 0]), float(z[0, 0]))
