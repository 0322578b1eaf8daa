"""Error certificates (reference bounds.py:45-140)
against golden values computed by the REFERENCE itself
(tests/golden/make_bounds_golden.py -> ref_bounds.npz)."""

import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_bounds.npz"))


@pytest.fixture(scope="module")
def rg():
    import paper_2404_09459_b200 as rg

    rg._native.require_device()
    return rg


def _spec(rg, c):
    a, b = GOLD[f"c{c}_alphas"], GOLD[f"c{c}_betas"]
    r = int(np.count_nonzero(b < 1e-10))
    za = int(np.count_nonzero(a < 1e-10))
    return rg.GsvSpectrum(a.copy(), b.copy(), r, a.size - r - za)


@pytest.mark.parametrize("c", [0, 1])
def test_projector_and_perturbation_bounds_match_reference(rg, c):
    pair = rg.GmpPair(GOLD[f"c{c}_g1"], GOLD[f"c{c}_g2"])
    pair_t = rg.GmpPair(GOLD[f"c{c}_g1t"], GOLD[f"c{c}_g2t"])
    assert math.isclose(pair.stack_norm2, float(GOLD[f"c{c}_stack_norm2"]), rel_tol=1e-12)
    assert math.isclose(pair.stack_pinv_norm, float(GOLD[f"c{c}_stack_pinv_norm"]),
                        rel_tol=1e-10)
    spec = _spec(rg, c)
    for k, os_, side, want in GOLD[f"c{c}_projector"]:
        got = rg.projector_bound(pair, spec, k=int(k), oversample=int(os_),
                                 which="first" if side == 0 else "second")
        assert math.isclose(got, want, rel_tol=1e-11, abs_tol=1e-300), (k, os_, side)
    got = rg.perturbation_bound(pair, pair_t)
    assert math.isclose(got, float(GOLD[f"c{c}_perturbation"]), rel_tol=1e-9)


@pytest.mark.parametrize("c", [0, 1])
@pytest.mark.parametrize("q", [0, 1, 2, 3])
def test_quantity_error_bounds_match_reference(rg, c, q):
    spec = _spec(rg, c)
    pre = f"c{c}_q{q}_"
    e = float(GOLD[pre + "e"])
    cert = rg.quantity_error_bounds(spec, e, eta=float(GOLD[f"c{c}_stack_norm2"]))
    assert cert.theta_bound == float(GOLD[pre + "theta_bound"])
    assert cert.vacuous == bool(GOLD[pre + "vacuous"])
    assert np.allclose(cert.p1_bounds, GOLD[pre + "p1"], rtol=1e-14, atol=0)
    assert np.allclose(cert.p2_bounds, GOLD[pre + "p2"], rtol=1e-14, atol=0)
    assert math.isclose(cert.d1_bound, float(GOLD[pre + "d1"]), rel_tol=1e-12)
    assert math.isclose(cert.d2_bound, float(GOLD[pre + "d2"]), rel_tol=1e-12)


def test_bound_validation_mirrors_reference(rg):
    pair = rg.GmpPair(GOLD["c0_g1"], GOLD["c0_g2"])
    spec = _spec(rg, 0)
    with pytest.raises(rg.ValidationError):
        rg.projector_bound(pair, spec, k=1, oversample=5)
    with pytest.raises(rg.ValidationError):
        rg.projector_bound(pair, spec, k=4, oversample=1)
    with pytest.raises(rg.ValidationError):
        rg.projector_bound(pair, spec, k=30, oversample=12)
    with pytest.raises(rg.ValidationError):
        rg.projector_bound(pair, spec, k=4, oversample=3, which="both")
    with pytest.raises(rg.ValidationError):
        rg.quantity_error_bounds(spec, -1.0)
    other = rg.GmpPair(GOLD["c1_g1"], GOLD["c1_g2"])
    with pytest.raises(rg.DimensionError):
        rg.perturbation_bound(pair, other)
