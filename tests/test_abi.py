"""The C-ABI library: loads without a GPU and exports every declared symbol."""

import ctypes

from paper_2404_09459_b200 import _native


def test_library_loads_and_versions():
    lib = _native.lib()
    assert b"sm_100a" in lib.rgsv_version()


def test_every_header_symbol_exported_and_typed():
    lib = _native.lib()
    syms = _native.header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, name


def test_workspace_queries_without_device():
    lib = _native.lib()
    assert lib.rgsv_sketch_workspace_bytes(20000, 1000, 60) > 20000 * 64 * 8
    assert lib.rgsv_small_gsvd_workspace_bytes(60, 60, 1000) > 120 * 1000 * 8
    assert lib.rgsv_svd_values_workspace_bytes(30, 40) >= 30 * 40 * 8


def test_argument_errors_are_reported_without_launch():
    lib = _native.lib()
    null = ctypes.c_void_p(0)
    # k > min(m, n) is the reference's max_cols ValidationError (rangefinder.py:88-91)
    rc = lib.rgsv_sketch_project(null, 10, 10, 10, null, 10, 11, 0, null, null, 10, null, null,
                                 null, null, 0, null)
    assert rc == _native.ERR_VALIDATION
    rc = lib.rgsv_sketch_project(null, 9, 10, 9, null, 10, 3, 0, null, null, 10, null, null,
                                 null, null, 0, null)
    assert rc == _native.ERR_DIMENSION  # odd leading dimension
    assert lib.rgsv_small_gsvd(null, 2, 0, null, 2, 0, 4, null, null, null, null, null, 0,
                               null) == _native.ERR_RANK
    assert lib.rgsv_comparative(null, null, null, 4, 0.5, null, null, null, null, null, null,
                                null, null, null, null) == _native.ERR_VALIDATION
    # tf32x3 entry points: N must be a multiple of 32 in [32, 320]; fp32
    # pitches a multiple of 4 elements; fp64 output pitch even
    assert lib.rgsv_tf32x3_gx(null, null, 64, null, null, 64, null, 48, 100, 48, 64,
                              null) == _native.ERR_DIMENSION
    assert lib.rgsv_tf32x3_gx(null, null, 66, null, null, 64, null, 64, 100, 64, 64,
                              null) == _native.ERR_DIMENSION
    assert lib.rgsv_tf32x3_gx(null, null, 64, null, null, 64, null, 352, 100, 352, 64,
                              null) == _native.ERR_DIMENSION
    assert lib.rgsv_tf32x3_gtq(null, null, 48, null, null, 64, null, 64, 48, 64, 100, null, 0,
                               null) == _native.ERR_DIMENSION
    assert lib.rgsv_f32_split(null, 8, 4, 16, null, 16, 0, null, null, 0,
                              null) == _native.ERR_DIMENSION
    assert lib.rgsv_f64_split_tf32(null, 8, 4, 8, null, null, 4, 4, null) == _native.ERR_DIMENSION


def test_error_mapping():
    import pytest

    from paper_2404_09459_b200 import errors

    for rc, exc in ((1, errors.DimensionError), (2, errors.ValidationError),
                    (3, errors.RankDeficiencyError), (4, errors.ConvergenceError),
                    (7, errors.DegenerateSpectrumError)):
        with pytest.raises(exc):
            _native.check(rc, "x")
    with pytest.raises(RuntimeError):
        _native.check(5, "x")
    assert errors.ConvergenceError.category == "numerical"
    assert errors.RecoveryError.category == "recovery"


def test_round2_entry_points_reject_bad_arguments_without_launch():
    """The round-2 entry points validate shapes before touching the device."""
    from paper_2404_09459_b200 import _native

    lib = _native.lib()
    null = None
    # rgsv_dense_qr: too many rows, bad leading dimensions, missing workspace
    assert lib.rgsv_dense_qr(null, 10, 1409, null, 0, 0, 10, null, 10, null, 0, 1, null, 0,
                             null) == 1
    assert lib.rgsv_dense_qr(null, 4, 8, null, 0, 0, 10, null, 8, null, 0, 1, null, 0,
                             null) == 2  # a1 is NULL -> validation error
    assert lib.rgsv_dense_qr_workspace_bytes(1409, 10) == 0
    # rgsv_spectrum_from_l_blocks: bad branch, classify_tol, ld < cols
    assert lib.rgsv_spectrum_from_l_blocks(null, 4, 2, null, 4, 2, 4, 8, 1e-10, 3, null, null,
                                           null, null, null, 0, null) == 1
    assert lib.rgsv_spectrum_from_l_blocks(null, 4, 2, null, 4, 2, 4, 8, 0.5, 0, null, null,
                                           null, null, null, 0, null) == 2
    assert lib.rgsv_spectrum_from_l_blocks(null, 3, 2, null, 4, 2, 4, 8, 1e-10, 0, null, null,
                                           null, null, null, 1 << 20, null) == 1
    # rgsv_svd_vectors_blocked / rgsv_gemm_gram_lower: leading dimensions
    assert lib.rgsv_svd_vectors_blocked(null, 3, 4, 8, null, 4, null, null, 8, null, 4, 0, null,
                                        null, null, 0, null) == 1
    assert lib.rgsv_gemm_gram_lower(null, 10, 16, 100, null, 8, null, 0, null) == 1
