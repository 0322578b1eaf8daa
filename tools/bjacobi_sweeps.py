"""Outer sweeps the blocked Jacobi (k_bjacobi) needs: reads the per-sweep
rotation flags it leaves in rgsv_svd_values' workspace (job 0 flags at
sync + 64, one int per sweep), for a few matrix families."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_09459_b200 import _native  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402

L = _native.lib()
st = dv.sp(torch.cuda.current_stream())
rng = np.random.default_rng(0)


def run(name, a):
    rows, cols = a.shape
    A = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    sv = torch.zeros(min(rows, cols), dtype=torch.float64, device="cuda")
    ints = torch.zeros(4, dtype=torch.int32, device="cuda")
    nb = int(L.rgsv_svd_values_workspace_bytes(rows, cols))
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _native.check(L.rgsv_svd_values(dv.vp(A), cols, rows, cols, dv.vp(sv), dv.vp(ints[:2]),
                                    dv.vp(ints[2:3]), dv.vp(ws), nb, st), "svd")
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    base = ((rows * cols * 8 + 255) // 256) * 256 + 64
    flags = ws[base: base + 60 * 4].view(torch.int32).cpu().numpy()
    ref = np.linalg.svd(a, compute_uv=False)
    print(f"{name:34s} {rows}x{cols}: {dt * 1e3:8.2f} ms, sweeps with rotations "
          f"{int(np.count_nonzero(flags))}, status {int(ints[2])}, "
          f"max err/s1 {np.max(np.abs(sv.cpu().numpy() - ref)) / ref[0]:.1e}", flush=True)


q = np.linalg.qr(rng.standard_normal((400, 200)))[0]
run("L1 of a 400x200 orthonormal Q", q[:200])
run("gaussian", rng.standard_normal((200, 200)))
run("gaussian", rng.standard_normal((120, 240)))
run("gaussian", rng.standard_normal((1000, 1000)))
u = np.linalg.qr(rng.standard_normal((300, 300)))[0]
run("graded 1..1e-12", (u * np.logspace(0, -12, 300)) @ np.linalg.qr(rng.standard_normal((300, 300)))[0].T)
