"""Per-phase clock64 breakdown of k_batch_chain (diagnostic build).

Builds /tmp/librgsv_b200_prof.so with -DRGSV_BATCH_PROFILE, loads it through
RGSV_LIB_PATH, runs a cfg3 batch and prints each phase's share of CTA time."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CSRC = os.path.join(ROOT, "paper_2404_09459_b200", "csrc")
OUT = "/tmp/librgsv_b200_prof.so"
srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".cu")]
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                       "-Xcompiler", "-fPIC", "-shared", "-DRGSV_BATCH_PROFILE", "-lcuda",
                       "-I", os.path.join(ROOT, "include"), "-o", OUT] + srcs)
os.environ["RGSV_LIB_PATH"] = OUT
import torch  # noqa: E402

import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS["cfg3"]
B = int(os.environ.get("B", 1024))
if os.environ.get("DATA", "cfg3") == "gauss":  # plain Gaussian matrices (well conditioned)
    gen = torch.Generator(device="cuda").manual_seed(0)
    g1 = torch.randn((B, cfg.m, cfg.n), generator=gen, device="cuda", dtype=torch.float64)
    g2 = torch.randn((B, cfg.p, cfg.n), generator=gen, device="cuda", dtype=torch.float64)
else:  # the bench's cfg3 data (workloads.py recipe: rank-8 signal + 1e-8 noise)
    import bench
    g1, g2 = bench.device_batch_pairs(cfg, B, 1000)
pairs = [(rg.device.DevMatrix(g1[j], cfg.m, cfg.n), rg.device.DevMatrix(g2[j], cfg.p, cfg.n))
         for j in range(B)]
plan = rg.device.small_batch_plan(B, cfg.n, cfg.k)
plan.set_pairs(pairs)
plan.set_seeds([2 * j for j in range(B)])
plan.launch(cfg.q, 1e-10)
torch.cuda.synchronize()
L = rg._native.lib()
buf = (ctypes.c_ulonglong * 24)()
L.rgsv_debug_batch_profile(buf, 1)
plan.launch(cfg.q, 1e-10)
torch.cuda.synchronize()
rg._native.check(L.rgsv_debug_batch_profile(buf, 0), "profile")
names = {0: "setup (Omega load, Y zero)", 1: "G X sketch pass (HBM)", 3: "G X later passes", 2: "G^T Q passes", 4: "gram",
         5: "gram reduce", 6: "chol", 7: "trsm", 8: "|G|^2 reduce", 10: "Z/B reduce",
         12: "tail (B write)"}
tot = sum(buf[i] for i in names)
nm = 2 * B
CS = int(os.environ.get("CS", 3))  # CTAs per cluster of the launched kernel (cfg3: 3)
for i, nmv in names.items():
    print(f"{nmv:28s} {buf[i] / tot * 100:5.1f}%  {buf[i] / nm / CS / 1.9e3:8.2f} us/matrix/CTA")
print(f"total {tot / nm / CS / 1.9e3:.1f} us per matrix-chain per CTA (clock ~1.9 GHz)")
print(f"chol calls {buf[15]}, near-identity fast path {buf[14]} "
      f"({buf[13] / max(buf[14], 1) / 1.9e3:.2f} us each incl. the check); "
      f"all chol phases {buf[6] / max(buf[15], 1) / 1.9e3:.2f} us per call")

print(f"shifted Gauss-Jordan (warp 0, per call): load+shift {buf[16] / max(buf[19], 1) / 1.9e3:.2f} us, "
      f"j-loop {buf[17] / max(buf[19], 1) / 1.9e3:.2f} us, store {buf[18] / max(buf[19], 1) / 1.9e3:.2f} us "
      f"({buf[19]} calls sampled)")
