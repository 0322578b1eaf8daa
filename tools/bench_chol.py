"""Time rgsv_chol_inv alone (CUDA events, 200 launches) for several sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402

L = _native.lib()
st = dv.sp(torch.cuda.current_stream())
for k in (16, 30, 60, 64, 120, 128, 240):
    kp = (k + 15) // 16 * 16
    x = np.random.default_rng(k).standard_normal((3 * k, k))
    G = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
    G[:k, :k] = torch.from_numpy(x.T @ x)
    linv = torch.zeros(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
    rinv = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    args = (dv.vp(G), k, kp, 1000, dv.vp(linv), dv.vp(rinv), None, dv.vp(status), st)
    for _ in range(5):
        L.rgsv_chol_inv(*args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        L.rgsv_chol_inv(*args)
    e1.record()
    e1.synchronize()
    print(f"chol k={k:4d} kp={kp:4d}: {e0.elapsed_time(e1) / 200 * 1e3:8.2f} us  status={int(status.item())}")

# reference points: tiny library launch and CUDA-graph replay of the Cholesky
x = torch.zeros((16, 16), dtype=torch.float64, device="cuda")
out = torch.zeros(4, dtype=torch.float64, device="cuda")
ws = torch.zeros(1024, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    L.rgsv_sumsq(dv.vp(x), 16, 16, 16, dv.vp(out), dv.vp(ws), 8 * 1024, st)
torch.cuda.synchronize()
e0.record()
for _ in range(200):
    L.rgsv_sumsq(dv.vp(x), 16, 16, 16, dv.vp(out), dv.vp(ws), 8 * 1024, st)
e1.record()
e1.synchronize()
print(f"sumsq (2 tiny kernels): {e0.elapsed_time(e1) / 200 * 1e3:8.2f} us")
for k in (16, 60, 120):
    kp = (k + 15) // 16 * 16
    xx = np.random.default_rng(k).standard_normal((3 * k, k))
    G = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
    G[:k, :k] = torch.from_numpy(xx.T @ xx)
    linv = torch.zeros(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
    rinv = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    g = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        L.rgsv_chol_inv(dv.vp(G), k, kp, 1000, dv.vp(linv), dv.vp(rinv), None, dv.vp(status),
                        dv.sp(s2))
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        cs = dv.sp(torch.cuda.current_stream())
        for _ in range(50):
            L.rgsv_chol_inv(dv.vp(G), k, kp, 1000, dv.vp(linv), dv.vp(rinv), None,
                            dv.vp(status), cs)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(4):
        g.replay()
    e1.record()
    e1.synchronize()
    print(f"graph chol k={k}: {e0.elapsed_time(e1) / 200 * 1e3:8.2f} us per launch")

# phase stamps of one k=60 Cholesky (thread 0 clock64 at each phase)
k, kp = 60, 64
xx = np.random.default_rng(1).standard_normal((200, k))
G = torch.zeros((kp, kp), dtype=torch.float64, device="cuda")
G[:k, :k] = torch.from_numpy(xx.T @ xx)
linv = torch.zeros(kp * kp + kp * (kp + 1), dtype=torch.float64, device="cuda")
prof = torch.zeros(64, dtype=torch.int64, device="cuda")
status = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    L.rgsv_debug_chol_profile(dv.vp(G), k, kp, dv.vp(linv), dv.vp(prof), dv.vp(status), st)
torch.cuda.synchronize()
p = prof.cpu().numpy()
base = p[0]
print("phase stamps (cycles from loop start): [diag done, panel done, update done] per block")
for jb in range(8):
    print(jb, p[2 + 4 * jb] - p[1 + 4 * jb], p[3 + 4 * jb] - p[2 + 4 * jb], p[4 + 4 * jb] - p[3 + 4 * jb])
print("total loop cycles", p[4 + 4 * 7] - base)
