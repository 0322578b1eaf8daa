"""Generate tests/golden/ref_bounds.npz by running the REFERENCE bounds
module (rgsv 0.1.0, bounds.py:45-140) here; the GPU box only loads the .npz.

    python tests/golden/make_bounds_golden.py

Cases: two real Gaussian pairs (reference.gaussian_matrix seeds 21..24,
shapes 60x30 / 45x30 and 80x40 / 70x40), their direct-method spectra, a
perturbed copy of each (1e-6 * Gaussian, seed + 100), and
  projector_bound(pair, spectrum, k, oversample, which) for several (k, p, side),
  perturbation_bound(pair, pair_tilde),
  quantity_error_bounds(spectrum, e, eta) for e in (1e-8, 1e-3, 0.2, 0.7).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import rgsv  # noqa: E402  (the reference)

out = {}
cases = [(60, 45, 30, 21), (80, 70, 40, 23)]
for ci, (m, p, n, sd) in enumerate(cases):
    g1 = rgsv.gaussian_matrix(m, n, sd)
    g2 = rgsv.gaussian_matrix(p, n, sd + 1)
    pair = rgsv.GmpPair(g1, g2)
    spec = rgsv.compute_gsv(pair, rgsv.GsvOptions(method="direct"))
    d1 = 1e-6 * rgsv.gaussian_matrix(m, n, sd + 100)
    d2 = 1e-6 * rgsv.gaussian_matrix(p, n, sd + 101)
    pair_t = rgsv.GmpPair(g1 + d1, g2 + d2)
    pre = f"c{ci}_"
    out[pre + "g1"], out[pre + "g2"] = g1, g2
    out[pre + "g1t"], out[pre + "g2t"] = g1 + d1, g2 + d2
    out[pre + "alphas"], out[pre + "betas"] = spec.alphas, spec.betas
    out[pre + "stack_norm2"] = np.array(pair.stack_norm2)
    out[pre + "stack_pinv_norm"] = np.array(pair.stack_pinv_norm)
    proj = []
    for k, os_, which in ((2, 2, "first"), (4, 3, "second"), (10, 5, "first"), (10, 5, "second")):
        proj.append([k, os_, 0 if which == "first" else 1,
                     rgsv.projector_bound(pair, spec, k=k, oversample=os_, which=which)])
    out[pre + "projector"] = np.array(proj)
    out[pre + "perturbation"] = np.array(rgsv.perturbation_bound(pair, pair_t))
    for ei, e in enumerate((1e-8, 1e-3, 0.2, 0.7)):
        cert = rgsv.quantity_error_bounds(spec, e, eta=pair.stack_norm2)
        q = f"{pre}q{ei}_"
        out[q + "e"] = np.array(e)
        out[q + "theta_bound"] = np.array(cert.theta_bound)
        out[q + "p1"], out[q + "p2"] = cert.p1_bounds, cert.p2_bounds
        out[q + "d1"], out[q + "d2"] = np.array(cert.d1_bound), np.array(cert.d2_bound)
        out[q + "vacuous"] = np.array(cert.vacuous)
np.savez(os.path.join(HERE, "ref_bounds.npz"), **out)
print("wrote", os.path.join(HERE, "ref_bounds.npz"), len(out), "arrays")
