"""ctypes binding of libcfb200.so (include/cfb200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2203_05027_b200.build``). There is no CPU fallback: if the
shared object is missing, or no CUDA device is visible when a plan is
created, the call raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_char_p, c_double, c_int, c_int32, c_int64, c_void_p

__all__ = ["lib", "LIB_PATH", "CfConfig", "CfReport", "CfChecks", "check", "CfError",
           "STATUS_NAMES", "TERM_MODES"]

LIB_PATH = os.environ.get("CF_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcfb200.so")

CF_OK, CF_EINVAL, CF_ECUDA, CF_ENOMEM, CF_EPROBLEM, CF_ESTATE = range(6)
STATUS_NAMES = ("running", "solved", "max_iters", "diverged")
TERM_MODES = ("osqp", "scs", "target")


class CfConfig(Structure):
    _fields_ = [
        ("mu", c_double),
        ("max_iters", c_int64),
        ("check_every", c_int64),
        ("term_mode", c_int32),
        ("reserved0", c_int32),
        ("eps_abs", c_double),
        ("eps_rel", c_double),
        ("b_inf", c_double),
        ("c_inf", c_double),
        ("scs_prim_bound", c_double),
        ("scs_dual_bound", c_double),
        ("eps_gap", c_double),
        ("target_prim_res", c_double),
        ("target_gap", c_double),
    ]


class CfReport(Structure):
    _fields_ = [
        ("iter", c_int64),
        ("status", c_int32),
        ("nonfinite", c_int32),
        ("prim_res_inf", c_double),
        ("prim_res_2", c_double),
        ("dual_res_inf", c_double),
        ("dual_res_2", c_double),
        ("stat_res_inf", c_double),
        ("stat_res_2", c_double),
        ("ax_inf", c_double),
        ("atl_inf", c_double),
        ("cone_gap", c_double),
        ("pobj", c_double),
        ("dobj", c_double),
        ("gap", c_double),
    ]


class CfChecks(Structure):
    _fields_ = [
        ("bad_row", c_int64),
        ("bad_col", c_int64),
        ("nonfinite_val", c_int64),
        ("zero_val", c_int64),
        ("duplicates", c_int64),
        ("nonfinite_b", c_int64),
        ("nonfinite_c", c_int64),
    ]


class CfError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_P = c_void_p
_D = POINTER(c_double)
_I64 = POINTER(c_int64)

# name -> (restype, argtypes); every symbol of include/cfb200.h
SIGNATURES = {
    "cf_last_error": (c_char_p, []),
    "cf_abi_version": (c_int, []),
    "cf_debug_guard_violations": (ctypes.c_longlong, []),
    "cf_device_count": (c_int, [POINTER(c_int)]),
    "cf_plan_create": (c_int, [c_int64, c_int64, c_int64, _P, _P, _P, _P, _P, c_int64, _P, c_int, _P,
                               POINTER(CfChecks), POINTER(c_void_p)]),
    "cf_plan_destroy": (c_int, [_P]),
    "cf_plan_info": (c_int, [_P, _I64, _I64, _I64, _I64, _I64, _I64, POINTER(c_int32)]),
    "cf_plan_set_rhs": (c_int, [_P, _P, _P, c_int]),
    "cf_plan_set_state": (c_int, [_P, c_double, _P, _P, _P, _P, _P, _P]),
    "cf_plan_set_export": (c_int, [_P, c_int]),
    "cf_plan_get_state": (c_int, [_P, _P, _P, _P, _P, _P, _P, _I64]),
    "cf_plan_iterate": (c_int, [_P, c_double, c_int64]),
    "cf_plan_report": (c_int, [_P, c_double, POINTER(CfReport)]),
    "cf_plan_solve": (c_int, [_P, POINTER(CfConfig), _P, _P, POINTER(CfReport), c_int64, _I64]),
    "cf_plan_trace": (c_int, [_P, c_int64, c_int64, POINTER(CfReport)]),
    "cf_apply_A": (c_int, [_P, _P, _P]),
    "cf_apply_At": (c_int, [_P, _P, _P]),
    "cf_apply_At_async": (c_int, [_P, _P, _P]),
    "cf_apply_At_cols": (c_int, [_P, _P, _P, c_int64, c_int64]),
    "cf_project": (c_int, [_P, _P, _P]),
    "cf_plan_last_timing": (c_int, [_P, _D, _I64, _D, _D, _I64]),
    "cf_plan_vector": (c_int, [_P, c_int, POINTER(c_void_p), _I64]),
    "cf_plan_column_counts": (c_int, [_P, _P]),
    "cf_plan_row_step": (c_int, [_P, c_double, c_int]),
    "cf_plan_row_parts": (c_int, [_P, _P]),
    "cf_column_update": (c_int, [c_int64, _P, _P, _P, _P, _P, _P, c_double, c_int64, _P, _P]),
    "cf_column_parts": (c_int, [c_int64, _P, _P, _P, _P, _P, _P, _P]),
    "cf_batch_solve": (c_int, [c_int64, _P, _P, c_int64, _P, _P, _P, _P, _P, c_int64, _P, _P, _P, _P, _P, _P, _P,
                               c_int64, POINTER(CfChecks), _D]),
    "cf_cluster_solve": (c_int, [c_int64, c_int64, c_int64, _P, _P, _P, _P, _P, c_int64, _P, _P, _P, _P, _P, _P, _P,
                                 c_int64, POINTER(CfChecks), _P, _D]),
    "cf_plan_set_profiling": (c_int, [_P, c_int]),
    "cf_plan_sync": (c_int, [_P]),
    "cf_plan_col_step": (c_int, [_P, c_double]),
    "cf_plan_row_norms": (c_int, [_P, _P, _P]),
    "cf_plan_set_row_norms": (c_int, [_P, _P, _P]),
    "cf_apply_A_async": (c_int, [_P, _P, _P]),
    "cf_plan_row_update": (c_int, [_P, c_double, c_int]),
    "cf_coneprob_open": (c_int, [c_char_p, c_char_p, c_int64, POINTER(c_void_p)]),
    "cf_coneprob_close": (None, [_P]),
    "cf_coneprob_header": (c_int, [_P, _I64, _I64, c_char_p, c_int64]),
    "cf_coneprob_sizes": (c_int, [_P, _P]),
    "cf_coneprob_body": (c_int, [_P, _P, _P, _P, _P, _P, c_int, _I64, c_char_p, c_int64]),
    "cf_format_double": (c_int, [c_double, c_char_p]),
    "cf_coneprob_write": (c_int, [c_char_p, c_int64, c_int64, c_int64, _P, _P, _P, _P, _P, c_int64, _P, c_int]),
    "cf_solution_write": (c_int, [c_char_p, c_char_p, _P, c_int64, _P, c_int64, c_int]),
    "cf_column_update_p2p": (c_int, [c_int64, _P, c_int32, _P, _P, _P, _P, _P, c_double, c_int64, _P, _P, c_int32,
                                     _P]),
    "cf_ipc_alloc": (c_int, [c_int64, POINTER(c_void_p), c_void_p]),
    "cf_ipc_free": (c_int, [_P]),
    "cf_ipc_open": (c_int, [c_void_p, POINTER(c_void_p)]),
    "cf_ipc_close": (c_int, [_P]),
    "cf_plan_bind_x": (c_int, [_P, _P]),
    "cf_plan_row_update_range": (c_int, [_P, c_double, c_int, c_int64, c_int64, _P]),
    "cf_plan_row_parts_range": (c_int, [_P, c_int64, c_int64, _P, _P]),
    "cf_plan_bind_h": (c_int, [_P, _P]),
    "cf_mc_supported": (c_int, [POINTER(c_int)]),
    "cf_mc_create": (c_int, [c_int64, c_int32, POINTER(c_void_p), POINTER(c_int)]),
    "cf_mc_import": (c_int, [c_int, c_int64, c_int32, POINTER(c_void_p)]),
    "cf_mc_add_device": (c_int, [_P]),
    "cf_mc_bind": (c_int, [_P, POINTER(c_void_p), POINTER(c_void_p)]),
    "cf_mc_destroy": (c_int, [_P]),
    "cf_column_update_nvls": (c_int, [c_int64, _P, _P, _P, _P, _P, _P, c_double, c_int64, _P, _P, _P]),
    "cf_mc_barrier": (c_int, [_P, _P, ctypes.c_uint32, _P]),
    "cf_gen_normal": (c_int, [ctypes.c_uint64, ctypes.c_uint64, c_int64, c_int64, _P, _P]),
    "cf_gen_cells": (c_int, [ctypes.c_uint64, c_int64, c_int64, c_int64, _P, _P]),
    "cf_gen_keys": (c_int, [ctypes.c_uint64, ctypes.c_uint64, c_int64, c_int64, _P, _P]),
}

_lib = None


def lib():
    """Load (once) and return the ctypes handle; raises if the library is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(nvcc, sm_100a). There is no CPU fallback."
            )
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.cf_abi_version() != 1:
            raise ImportError("libcfb200.so ABI version mismatch; rebuild it")
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().cf_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == CF_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == CF_EINVAL:
        raise ValueError(msg)
    if rc == CF_ENOMEM:
        raise MemoryError(msg)
    raise CfError(rc, msg)


def device_count() -> int:
    n = c_int(0)
    lib().cf_device_count(ctypes.byref(n))
    return int(n.value)
