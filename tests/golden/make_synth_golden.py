"""Generate tests/golden/ref_synth.npz and tests/golden/io/bench_records.{csv,json}
by running the REFERENCE's generator, timing harness and report writer
(rgsv 0.1.0: synthetic.py:63-112, bench.py:82-136, io.py:171-178,236-245) here;
the tests only read the committed files.

    python tests/golden/make_synth_golden.py

ref_synth.npz: for each real-field case (m, p, n, rank_frac, seed) the
reference's g1, g2, true alphas / betas, r, s and condition_r.
bench_records.*: the reference's serialization of two fixed BenchRecords
(one direct with residuals None, one randomized).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import rgsv  # noqa: E402  (the reference)
from rgsv.bench import BenchRecord  # noqa: E402

CASES = [(40, 30, 12, 0.75, 3), (8, 9, 12, 1.0, 1), (200, 150, 64, 0.6, 7), (1500, 40, 24, 0.9, 11)]

out = {"cases": np.array(CASES, dtype=np.float64)}
for i, (m, p, n, frac, seed) in enumerate(CASES):
    res = rgsv.synth_gmp(rgsv.SynthSpec(m=m, p=p, n=n, rank_frac=frac, seed=seed, field="real"))
    out[f"g1_{i}"] = res.pair.g1
    out[f"g2_{i}"] = res.pair.g2
    out[f"alphas_{i}"] = res.true_spectrum.alphas
    out[f"betas_{i}"] = res.true_spectrum.betas
    out[f"rs_{i}"] = np.array([res.true_spectrum.r, res.true_spectrum.s])
    out[f"cond_{i}"] = np.array(res.condition_r)
np.savez_compressed(os.path.join(HERE, "ref_synth.npz"), **out)

records = [
    BenchRecord("direct", 0, 0.012345678901234567, 0.0, 0.0, None, None, 44, 40, 24, 20, 12),
    BenchRecord("randomized", 1, 1.5e-3, 3.25e-15, 1.0 / 3.0, 2.5e-11, 1e-300, 12, 12, 24, 20, 12),
]
for fmt in ("csv", "json"):
    rgsv.write_report(records, os.path.join(HERE, "io", f"bench_records.{fmt}"), fmt)
print("wrote ref_synth.npz, io/bench_records.{csv,json}")
