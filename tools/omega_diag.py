import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2404_09459_b200 import device as dv
seeds = list(range(0, 8192, 2))
om = dv.omega_device(64, 16, seeds).cpu().numpy()
for i, seed in enumerate(seeds):
    ref = np.random.default_rng(seed).standard_normal((64, 16))
    got = om[i, :16, :64].T
    bad = np.nonzero(got != ref)
    for r, c in zip(*bad):
        e = r * 16 + c
        print(seed, e, repr(ref[r, c]), repr(got[r, c]), 'ulps', int(abs(ref[r,c].view(np.int64) - got[r,c].view(np.int64))))
