"""ctypes binding of the in-tree C-ABI library (include/htlr_b200.h).

The library is loaded from this package directory only; if it is missing the
import fails loudly (there is no CPU fallback).  Error codes map to the
reference's exception types: negative -> ValueError, positive ->
RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_htlr_b200.so")

HTLR_KERNEL_GAUSSIAN = 0
HTLR_KERNEL_SLP2D = 1
HTLR_KERNEL_SLP3D = 2
HTLR_RULE_WEAK = 0
HTLR_RULE_STRONG = 1


class HtlrDesc(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("leaf_side_max", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("rule", ctypes.c_int32),
        ("eta", ctypes.c_double),
        ("kernel", ctypes.c_int32),
        ("sigma", ctypes.c_double),
        ("scale", ctypes.c_double),
        ("quad_q", ctypes.c_int32),
        ("corner_subdivision", ctypes.c_int32),
        ("coeff_const", ctypes.c_double),
        ("grid_kind", ctypes.c_int32),
        ("amplitude", ctypes.c_double),
    ]


# (name, restype, argtypes) for every symbol declared in include/htlr_b200.h
_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double
SYMBOLS = [
    ("htlr_plan_create", ctypes.c_int, [ctypes.POINTER(HtlrDesc), ctypes.c_int, ctypes.POINTER(_P)]),
    ("htlr_plan_destroy", ctypes.c_int, [_P]),
    ("htlr_build_lists", ctypes.c_int, [_P]),
    ("htlr_tree_info", ctypes.c_int, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32), ctypes.POINTER(_I64),
                                      ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    ("htlr_export_lists", ctypes.c_int, [_P, _P, _I64]),
    ("htlr_set_coeff", ctypes.c_int, [_P, _P]),
    ("htlr_construct", ctypes.c_int, [_P, _P]),
    ("htlr_matvec", ctypes.c_int, [_P, _P, _P, _I64, _P]),
    ("htlr_matvec_host", ctypes.c_int, [_P, _P, _P, _I64, _P]),
    ("htlr_matvec_remote_begin", ctypes.c_int, [_P, _P, _I64, _P]),
    ("htlr_matvec_remote_finish", ctypes.c_int, [_P, _P, _P, _I64, _P]),
    ("htlr_set_lowrank", ctypes.c_int, [_P, _I32]),
    ("htlr_set_shard", ctypes.c_int, [_P, _I32, _I32]),
    ("htlr_set_zslab", ctypes.c_int, [_P, _I32, _I32]),
    ("htlr_kernel_pairs_masked", ctypes.c_int, [_I32, ctypes.c_double, ctypes.c_double, _I32, _P, _I64, _P, _P]),
    ("htlr_mode_product", ctypes.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P]),
    ("htlr_gemm", ctypes.c_int, [_P, _P, _I64, _I64, _I64, _P]),
    ("htlr_kron", ctypes.c_int, [_P, _I64, _I64, _P, _I64, _I64, _P]),
    ("htlr_qr", ctypes.c_int, [_P, _I64, _I64, _P, _P]),
    ("htlr_exchange_kind", ctypes.c_int, [_P]),
    ("htlr_shard_info", ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                                       ctypes.POINTER(_D)]),
    ("htlr_exchange_info", ctypes.c_int, [_P, _I64, ctypes.POINTER(_I64), _P, _I64]),
    ("htlr_bind_exchange", ctypes.c_int, [_P, _I64, _P, _I64]),
    ("htlr_matvec_local", ctypes.c_int, [_P, _P, _I64, _P]),
    ("htlr_matvec_remote", ctypes.c_int, [_P, _P, _P, _I64, _P]),
    ("htlr_reduce_info", ctypes.c_int, [_P, _I64, ctypes.POINTER(_I64), _P, _I64]),
    ("htlr_bind_reduce", ctypes.c_int, [_P, _I64, _P, _I64]),
    ("htlr_matvec_contract", ctypes.c_int, [_P, _P, _I64, _P]),
    ("htlr_matvec_expand", ctypes.c_int, [_P, _P, _P, _I64, _P]),
    ("htlr_diag_value", ctypes.c_int, [_P, ctypes.POINTER(_D)]),
    ("htlr_export_block", ctypes.c_int, [_P, _I64, _P, _I64, _P, _I64, _P]),
    ("htlr_storage", ctypes.c_int, [_P, _P]),
    ("htlr_formulation", ctypes.c_int, [_P]),
    ("htlr_leaf_pass", ctypes.c_int, [_P]),
    ("htlr_cell_average", ctypes.c_int, [_I32, _D, _D, _I32, _D, _I32, _I32, ctypes.c_int, ctypes.POINTER(_D)]),
    ("htlr_exact_rows", ctypes.c_int, [_P, _P, _I64, _P, _P, _P]),
    ("htlr_set_graphs", ctypes.c_int, [_P, _I32]),
    ("htlr_overlap_areas", ctypes.c_int, [_P, _P, _I64, _I32, _P, _P]),
    ("htlr_cheb_nodes", ctypes.c_int, [_D, _D, _I32, _P]),
    ("htlr_lagrange_matrix", ctypes.c_int, [_P, _I64, _P, _I32, _P]),
    ("htlr_kernel_pairs", ctypes.c_int, [_I32, _D, _D, _I32, _P, _I64, _P, _I64, _P]),
    ("htlr_csr_spmv", ctypes.c_int, [_P, _P, _P, _I64, _P, _P, _P]),
    ("htlr_profile_enable", ctypes.c_int, [_P, _I32]),
    ("htlr_profile_read", ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I64, ctypes.POINTER(_I64)]),
    ("htlr_last_launch_count", _I64, [_P]),
    ("htlr_last_error", ctypes.c_char_p, []),
]

_lib = None


def lib():
    """Load (once) and return the C-ABI library."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2508_05958_b200.build` "
                "(there is no CPU fallback for the HTLR hot path)")
        handle = ctypes.CDLL(LIB_PATH)
        for name, res, args in SYMBOLS:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().htlr_last_error().decode(errors="replace")
    if rc < 0:
        raise ValueError(msg)
    raise RuntimeError(msg)
