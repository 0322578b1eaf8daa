"""Relative Frobenius error of the 3xTF32 tcgen05 GEMMs vs fp64, by K
(diagnostic for the accumulation error of the TMEM fp32 accumulator)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2404_09459_b200 as rg

t = rg.tf32.TF32Ops()
L = rg._native.lib()
for M, N in ((512, 288), (512, 64)):
    for K in (64, 256, 1024, 4096, 8192, 32768):
        rng = np.random.default_rng(K)
        g32 = rng.standard_normal((M, K)).astype(np.float32)
        xt = rng.standard_normal((N, K))
        g = rg.device.to_device(torch.from_numpy(g32).cuda(), "g", keep_f32=True)
        lo, _ = t.split_big(g)
        xh, xl = t.split_small(torch.from_numpy(xt).cuda(), N, K, K)
        y = torch.zeros((M, N), dtype=torch.float64, device="cuda")
        t.gx(g, lo, xh, xl, y, M, N, K)
        ref = g32.astype(np.float64) @ xt.T
        e = np.linalg.norm(y.cpu().numpy() - ref) / np.linalg.norm(ref)
        # fp32 (numpy sgemm) for comparison
        r32 = (g32 @ xt.T.astype(np.float32)).astype(np.float64)
        e32 = np.linalg.norm(r32 - ref) / np.linalg.norm(ref)
        # positive data (no cancellation): bias check
        gp = np.abs(g32); xp = np.abs(xt)
        g2 = rg.device.to_device(torch.from_numpy(gp).cuda(), "g", keep_f32=True)
        lo2, _ = t.split_big(g2)
        xh2, xl2 = t.split_small(torch.from_numpy(xp).cuda(), N, K, K)
        t.gx(g2, lo2, xh2, xl2, y, M, N, K)
        refp = gp.astype(np.float64) @ xp.T
        ep = np.linalg.norm(y.cpu().numpy() - refp) / np.linalg.norm(refp)
        sgn = np.mean(np.sign(y.cpu().numpy() - refp))
        print(f"M={M} N={N} K={K}: gx rel err {e:.2e} (numpy fp32 sgemm {e32:.2e}); positive data {ep:.2e} mean sign {sgn:+.2f}", flush=True)
