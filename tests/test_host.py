"""Host-side logic of the drop-in API (no device needed)."""

import math

import numpy as np
import pytest

from paper_2404_09459_b200 import (
    ExtractionConfig,
    GsvOptions,
    GsvSpectrum,
    ValidationError,
    DimensionError,
    classify_spectrum,
    gaussian_matrix,
)
from paper_2404_09459_b200.rangefinder import single_block_width
from paper_2404_09459_b200.workloads import CONFIGS, make_pair


def test_config_validation_mirrors_reference():
    with pytest.raises(ValidationError):
        ExtractionConfig(tol=0.0)
    with pytest.raises(ValidationError):
        ExtractionConfig(blocksize=0)
    with pytest.raises(ValidationError):
        ExtractionConfig(trim_tol=-1e-3)
    with pytest.raises(ValidationError):
        ExtractionConfig(max_cols=0)
    with pytest.raises(ValidationError):
        ExtractionConfig(power_iters=-1)
    with pytest.raises(ValidationError):
        GsvOptions(classify_tol=0.5)
    with pytest.raises(ValidationError):
        GsvOptions(method="magic")


def test_single_block_detection():
    fixed = ExtractionConfig.fixed_rank(30, seed=0, power_iters=1)
    assert single_block_width(fixed, 2000, 200) == 30
    assert single_block_width(ExtractionConfig(blocksize=500, trim_tol=0.0), 50, 200) == 200
    # adaptive default (trim on, several blocks) is not a single block
    assert single_block_width(ExtractionConfig(), 2000, 200) is None
    assert single_block_width(ExtractionConfig(blocksize=10, max_cols=30, trim_tol=0.0),
                              100, 50) is None


def test_spectrum_invariants():
    with pytest.raises(ValidationError):
        GsvSpectrum(np.array([0.9, 0.5]), np.array([0.9, 0.5]), r=0, s=2)
    with pytest.raises(ValidationError):
        GsvSpectrum(np.array([0.5, 0.9]), np.sqrt(1 - np.array([0.5, 0.9]) ** 2), r=0, s=2)
    with pytest.raises(ValidationError):
        GsvSpectrum(np.array([1.0, 0.5]), np.array([1e-13, math.sqrt(0.75)]), r=1, s=1)
    with pytest.raises(DimensionError):
        GsvSpectrum(np.array([]), np.array([]), r=0, s=0)
    spec = GsvSpectrum(np.array([1.0, 0.6, 0.0]), np.array([0.0, 0.8, 1.0]), 1, 1)
    assert spec.n == 3


def test_classify_snaps_in_place():
    a = np.array([1.0 - 1e-13, 0.6, 1e-12])
    b = np.array([5e-13, 0.8, 1.0 - 1e-14])
    assert classify_spectrum(a, b, 1e-10) == (1, 1)
    assert a[0] == 1.0 and b[0] == 0.0 and a[2] == 0.0 and b[2] == 1.0
    with pytest.raises(ValidationError):
        classify_spectrum(np.array([1.0]), np.array([0.0]), classify_tol=0.5)


def test_gaussian_matrix_reference_convention():
    g = gaussian_matrix(5, 3, 7)
    assert np.array_equal(g, np.random.default_rng(7).standard_normal((5, 3)))
    c = gaussian_matrix(4, 2, 1, "complex")
    assert np.iscomplexobj(c)
    with pytest.raises(ValidationError):
        gaussian_matrix(2, 2, 0, "quaternion")
    with pytest.raises(DimensionError):
        gaussian_matrix(0, 2, 0)


def test_workload_generator():
    cfg = CONFIGS["cfg0"]
    g1, g2 = make_pair(cfg)
    assert g1.shape == (2000, 200) and g2.shape == (1500, 200)
    h1, _ = make_pair(cfg)
    assert np.array_equal(g1, h1)
    s = np.linalg.svd(g1, compute_uv=False)
    assert s[19] > 1e3 * s[20]  # rank-20 signal over 1e-8 noise
    assert CONFIGS["cfg1"].flops == 2.0 * 36000 * 1000 * 60 * 6
    assert CONFIGS["cfg3"].batch == 4096
