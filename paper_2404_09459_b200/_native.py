"""ctypes binding of the in-tree C-ABI library ``librgsv_b200.so``.

The library is the product: there is no CPU fallback. ``lib()`` raises
when the library is missing, and ``require_device()`` raises when no
sm_100 GPU is visible, so a misconfigured box fails loudly instead of
computing something else.
"""

from __future__ import annotations

import ctypes
import os
import re

from .errors import (
    ConvergenceError,
    DegenerateSpectrumError,
    DimensionError,
    RankDeficiencyError,
    ValidationError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RGSV_LIB_PATH") or os.path.join(HERE, "librgsv_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "rgsv_b200.h")

OK, ERR_DIMENSION, ERR_VALIDATION, ERR_RANK, ERR_CONVERGENCE, ERR_CUDA, ERR_WORKSPACE, \
    ERR_DEGENERATE = range(8)
ST_CHOL, ST_NONFINITE, ST_JACOBI, ST_CLASSIFY, ST_DEGENERATE, ST_NOT_NORMALIZED = (
    0x1, 0x2, 0x4, 0x8, 0x10, 0x20)
ST_OMEGA_SHORT = 0x40
ST_SPECTRUM = 0x80  # GsvSpectrum invariant violated (k_batch_small)

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_sz = ctypes.c_size_t
_d = ctypes.c_double

# name -> (restype, argtypes); must match include/rgsv_b200.h
SIGNATURES = {
    "rgsv_version": (ctypes.c_char_p, []),
    "rgsv_device_cc": (_i32, []),
    "rgsv_launch_count": (ctypes.c_longlong, []),
    "rgsv_omega_workspace_bytes": (_sz, [_i32, _i64, _i32]),
    "rgsv_omega_generate": (_i32, [_p, _i32, _i64, _i32, _p, _i64, _i64, _p, _p, _sz, _p]),
    "rgsv_omega_workspace_bytes_at": (_sz, [_i32, _i64, _i32, _i64]),
    "rgsv_omega_generate_at": (_i32, [_p, _i32, _i64, _i32, _i64, _p, _i64, _i64, _p, _p, _sz,
                                      _p]),
    "rgsv_householder_qr": (_i32, [_p, _i64, _i32, _i32, _p, _i64, _p, _p, _p]),
    "rgsv_axpy": (_i32, [_p, _i64, _p, _i64, _i32, _i32, _d, _p]),
    "rgsv_orth_complete": (_i32, [_p, _i64, _i32, _i32, _i32, _p, _i64, _p, _p, _p]),
    "rgsv_svd_vectors_blocked_workspace_bytes": (_sz, [_i32]),
    "rgsv_svd_vectors_blocked": (_i32, [_p, _i64, _i32, _i32, _p, _i64, _p, _p, _i64, _p, _i64,
                                        _i32, _p, _p, _p, _sz, _p]),
    "rgsv_svd_vectors": (_i32, [_p, _i64, _i32, _i32, _p, _i64, _p, _p, _i64, _p, _i64, _i32,
                                _p, _p, _p]),
    "rgsv_transpose": (_i32, [_p, _i64, _p, _i64, _i32, _i32, _p]),
    "rgsv_batch_supported": (_i32, [_i32, _i64, _i32]),
    "rgsv_debug_batch_profile": (_i32, [_p, _i32]),
    "rgsv_batch_workspace_bytes": (_sz, [_i32, _i64, _i32]),
    "rgsv_batch_gsvd": (_i32, [_p, _i32, _i32, _i64, _i32, _i32, _p, _d, _p, _p, _p, _p, _p, _p,
                               _sz, _p]),
    "rgsv_scale_cols": (_i32, [_p, _i64, _i32, _i32, _p, _p]),
    "rgsv_convert_f32": (_i32, [_p, _i64, _i64, _i64, _p, _i64, _p]),
    "rgsv_sketch_workspace_bytes": (_sz, [_i64, _i64, _i32]),
    "rgsv_sketch_project": (_i32, [_p, _i64, _i64, _i64, _p, _i64, _i32, _i32, _p, _p, _i64, _p,
                                   _p, _p, _p, _sz, _p]),
    "rgsv_sketch_project_sharded": (_i32, [_p, _i64, _i64, _i64, _i64, _p, _i64, _i32, _i32, _p,
                                           _p, _i64, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "rgsv_nccl_version": (_i32, []),
    "rgsv_nccl_get_unique_id": (_i32, [_p]),
    "rgsv_nccl_comm_init": (_i32, [_p, _i32, _p, _i32]),
    "rgsv_nccl_comm_destroy": (_i32, [_p]),
    "rgsv_nccl_allreduce": (_i32, [_p, _i64, _p, _p]),
    "rgsv_nccl_broadcast": (_i32, [_p, _i64, _i32, _p, _p]),
    "rgsv_small_gsvd_workspace_bytes": (_sz, [_i32, _i32, _i64]),
    "rgsv_small_gsvd": (_i32, [_p, _i64, _i32, _p, _i64, _i32, _i64, _p, _p, _p, _p, _p, _sz,
                               _p]),
    "rgsv_dense_qr_workspace_bytes": (_sz, [_i32, _i32]),
    "rgsv_dense_qr": (_i32, [_p, _i64, _i32, _p, _i64, _i32, _i32, _p, _i64, _p, _i64, _i32, _p,
                             _sz, _p]),
    "rgsv_comparative": (_i32, [_p, _p, _p, _i64, _d, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "rgsv_spectrum_from_l_blocks_workspace_bytes": (_sz, [_i32, _i32, _i32, _i64]),
    "rgsv_spectrum_from_l_blocks": (_i32, [_p, _i64, _i32, _p, _i64, _i32, _i32, _i64, _d, _i32,
                                           _p, _p, _p, _p, _p, _sz, _p]),
    "rgsv_spectrum_quantities": (_i32, [_p, _p, _i64, _i32, _p, _p, _p, _p, _p, _p, _p]),
    "rgsv_entropy": (_i32, [_p, _i64, _p, _p]),
    "rgsv_svd_values_workspace_bytes": (_sz, [_i32, _i32]),
    "rgsv_svd_values": (_i32, [_p, _i64, _i32, _i32, _p, _p, _p, _p, _sz, _p]),
    "rgsv_gemm_gx": (_i32, [_p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _p, _sz, _p]),
    "rgsv_gemm_gram_lower": (_i32, [_p, _i64, _i64, _i64, _p, _i64, _p, _sz, _p]),
    "rgsv_gemm_gtq": (_i32, [_p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _p, _sz, _p]),
    "rgsv_chol_inv": (_i32, [_p, _i32, _i32, _i64, _p, _p, _p, _p, _p]),
    "rgsv_debug_householder_profile": (_i32, [_p, _i64, _i32, _p, _i64, _i32, _p, _i64, _p, _p]),
    "rgsv_debug_dense_qr_profile": (_i32, [_p, _i64, _i32, _i32, _p, _p, _sz, _p, _p]),
    "rgsv_debug_chol_profile": (_i32, [_p, _i32, _i32, _p, _p, _p, _p]),
    "rgsv_sumsq": (_i32, [_p, _i64, _i64, _i64, _p, _p, _sz, _p]),
    "rgsv_f32_split": (_i32, [_p, _i64, _i64, _i64, _p, _i64, _i32, _p, _p, _sz, _p]),
    "rgsv_f64_split_tf32": (_i32, [_p, _i64, _i64, _i64, _p, _p, _i64, _i64, _p]),
    "rgsv_tf32x3_gx": (_i32, [_p, _p, _i64, _p, _p, _i64, _p, _i64, _i64, _i64, _i64, _p]),
    "rgsv_tf32x3_gtq": (_i32, [_p, _p, _i64, _p, _p, _i64, _p, _i64, _i64, _i64, _i64, _p, _sz,
                               _p]),
    "rgsv_tf32_config": (_i32, [_i32, _i32, _i32, _i32]),
}

_LIB = None


def header_symbols() -> list[str]:
    """Entry points declared in include/rgsv_b200.h (for the export test)."""
    with open(HEADER) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(rgsv_[a-z0-9_]+)\s*\(", text)))


def lib():
    """Load and type the library (no device needed)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -m paper_2404_09459_b200.build` "
                "(the sm_100a kernels are the only implementation, there is no CPU fallback)")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    return _LIB


def check(rc: int, what: str) -> None:
    """Map a C-ABI return code onto the reference exception classes."""
    if rc == OK:
        return
    msg = f"{what} failed (rgsv_b200 code {rc})"
    if rc == ERR_DIMENSION:
        raise DimensionError(msg)
    if rc == ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == ERR_RANK:
        raise RankDeficiencyError(msg)
    if rc == ERR_CONVERGENCE:
        raise ConvergenceError(msg)
    if rc == ERR_DEGENERATE:
        raise DegenerateSpectrumError(msg)
    raise RuntimeError(msg)


_DEVICE_OK = False


def require_device():
    """The hot path runs only on an sm_100 (B200) GPU; fail loudly otherwise."""
    global _DEVICE_OK
    if _DEVICE_OK:
        return
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2404_09459_b200 needs a CUDA (sm_100a) device: the rGSVD hot path is "
            "implemented only as B200 kernels and has no CPU fallback")
    torch.cuda.init()
    cc = lib().rgsv_device_cc()
    if cc < 100 or cc >= 110:
        raise RuntimeError(f"librgsv_b200 is built for sm_100a; current device reports cc={cc}")
    _DEVICE_OK = True
