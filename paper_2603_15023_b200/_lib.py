"""ctypes declaration of libpac.so (include/pac.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PAC_LIB") or os.path.join(HERE, "libpac.so")  # PAC_LIB: A/B experiments

PAC_M = 64
PAC_MAX_AGGS = 8
PAC_MAX_KEYS = 4

PAC_OK, PAC_E_INVAL, PAC_E_CAPACITY, PAC_E_WORKSPACE, PAC_E_CUDA, PAC_E_OVERFLOW, PAC_E_MERGE = range(7)
STATUS_NAMES = {0: "PAC_OK", 1: "PAC_E_INVAL", 2: "PAC_E_CAPACITY", 3: "PAC_E_WORKSPACE",
                4: "PAC_E_CUDA", 5: "PAC_E_OVERFLOW", 6: "PAC_E_MERGE"}

COUNT, SUM_I64, SUM_F64, AVG_F64, MIN_F64, MAX_F64 = range(6)


class PacError(RuntimeError):
    def __init__(self, fn: str, rc: int):
        super().__init__(f"{fn} returned {STATUS_NAMES.get(rc, rc)}")
        self.rc = rc


class AggSpec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("d_values", ctypes.c_void_p)]


class KeyCol(ctypes.Structure):
    _fields_ = [("d_col", ctypes.c_void_p), ("elem_bytes", ctypes.c_int32)]


class WVec(ctypes.Structure):
    _fields_ = [("d_y", ctypes.c_void_p), ("d_presence", ctypes.c_void_p), ("scalar", ctypes.c_double)]


OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_MIN, OP_MAX = range(6)
CMP_LT, CMP_LE, CMP_GT, CMP_GE, CMP_EQ = range(5)
PAC_CMP_INDEX_WORDS = 130


class Table(ctypes.Structure):
    _fields_ = [("d_num_groups", ctypes.c_void_p), ("d_status", ctypes.c_void_p),
                ("d_group_key", ctypes.c_void_p), ("d_rows", ctypes.c_void_p),
                ("d_presence", ctypes.c_void_p), ("d_count", ctypes.c_void_p),
                ("d_world", ctypes.c_void_p * PAC_MAX_AGGS), ("m", ctypes.c_int32)]


_P = ctypes.c_void_p
_lib = None


def lib() -> ctypes.CDLL:
    """Loads libpac.so.  There is no fallback: a missing library is an error."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing; run `python build.py` (or __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "pac_session_create": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_double, ctypes.POINTER(_P)]),
        "pac_session_destroy": (ctypes.c_int, [_P]),
        "pac_session_create_m": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_double, ctypes.c_int32, ctypes.POINTER(_P)]),
        "pac_session_worlds": (ctypes.c_int32, [_P]),
        "pac_mask128": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_uint64, _P, _P]),
        "pac_agg_workspace_size128": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                                     _P]),
        "pac_agg_grouped128": (ctypes.c_int, [_P, _P, ctypes.c_uint64, _P, ctypes.c_int, _P, ctypes.c_int,
                                              ctypes.c_int64, _P, ctypes.c_int64, _P, ctypes.c_size_t, _P]),
        "pac_session_query": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P]),
        "pac_session_set_posterior": (ctypes.c_int, [_P, _P]),
        "pac_session_posterior_device": (_P, [_P]),
        "pac_mask": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_uint64, _P, _P]),
        "pac_agg_workspace_size": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int64, _P]),
        "pac_agg_workspace_size_rows": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _P]),
        "pac_agg_grouped": (ctypes.c_int, [_P, _P, ctypes.c_uint64, _P, ctypes.c_int, _P, ctypes.c_int,
                                           ctypes.c_int64, _P, ctypes.c_int64, _P, ctypes.c_size_t, _P]),
        "pac_table_check": (ctypes.c_int, [_P, _P, _P]),
        "pac_table_rederive_presence": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int64, _P]),
        "pac_table_remap": (ctypes.c_int, [_P, _P, ctypes.c_int64, _P, ctypes.c_int, ctypes.c_int64, _P, _P]),
        "pac_finalize_workspace_size": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int, _P]),
        "pac_finalize": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, _P, _P, _P,
                                        _P, _P, ctypes.c_size_t, _P]),
        "pac_posterior_update": (ctypes.c_int, [_P, _P, ctypes.c_double, ctypes.c_double, _P]),
        "pac_world_vector": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _P, _P, _P]),
        "pac_lift": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_int64, _P, _P, _P]),
        "pac_lift_cmp": (ctypes.c_int, [ctypes.c_int, _P, _P, ctypes.c_int64, _P, _P]),
        "pac_noised_y_workspace_size": (ctypes.c_int, [ctypes.c_int64, _P]),
        "pac_noised_y": (ctypes.c_int, [_P, _P, _P, ctypes.c_int64, ctypes.c_uint32, _P, _P, _P, _P,
                                        ctypes.c_size_t, _P]),
        "pac_cmp_index": (ctypes.c_int, [_P, _P, ctypes.c_int64, _P, _P]),
        "pac_select": (ctypes.c_int, [_P, _P, _P, ctypes.c_int64, _P, _P]),
        "pac_select_cmp": (ctypes.c_int, [ctypes.c_int, _P, _P, _P, _P, ctypes.c_int64, _P, _P]),
        "pac_filter": (ctypes.c_int, [_P, _P, ctypes.c_int64, ctypes.c_uint32, _P, _P]),
        "pac_filter_cmp": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, ctypes.c_int64, ctypes.c_uint32, _P, _P]),
        "pac_join_table_bytes": (ctypes.c_int, [ctypes.c_int64, _P]),
        "pac_join_build": (ctypes.c_int, [_P, _P, ctypes.c_int64, _P, ctypes.c_size_t, _P]),
        "pac_join_table_status": (ctypes.c_int, [_P, _P]),
        "pac_join_mask": (ctypes.c_int, [_P, ctypes.c_int, _P, ctypes.c_int64, ctypes.c_uint64, _P, _P, _P]),
        "pac_launch_count": (ctypes.c_uint64, []),
        "pac_profile_enable": (ctypes.c_int, [ctypes.c_int]),
        "pac_profile_read": (ctypes.c_int, [_P, _P]),
        "pac_profile_last_kernel": (ctypes.c_char_p, []),
        "pac_merge_sizes": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int64, _P, _P, _P]),
        "pac_approx_sum_workspace_size": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, _P]),
        "pac_approx_sum": (ctypes.c_int, [_P, _P, ctypes.c_uint64, _P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64,
                                          _P, _P, _P, ctypes.c_size_t, _P]),
        "pac_merge_pack": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int64, _P, _P, _P, _P]),
        "pac_merge_unpack": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int64, _P, _P, _P, _P]),
        "pac_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(fn: str, rc: int) -> None:
    if rc != PAC_OK:
        raise PacError(fn, rc)


def exported_symbols() -> list:
    return ["pac_session_create", "pac_session_create_m", "pac_session_worlds", "pac_mask128",
            "pac_agg_workspace_size128", "pac_agg_grouped128", "pac_session_destroy", "pac_session_query", "pac_session_set_posterior",
            "pac_session_posterior_device", "pac_mask", "pac_agg_workspace_size", "pac_agg_workspace_size_rows", "pac_agg_grouped",
            "pac_table_check", "pac_table_rederive_presence", "pac_table_remap",
            "pac_finalize_workspace_size", "pac_finalize", "pac_posterior_update", "pac_world_vector",
            "pac_lift", "pac_lift_cmp", "pac_noised_y_workspace_size", "pac_noised_y", "pac_cmp_index",
            "pac_select", "pac_select_cmp", "pac_filter", "pac_filter_cmp", "pac_join_table_bytes",
            "pac_join_build", "pac_join_table_status", "pac_join_mask", "pac_launch_count",
            "pac_profile_enable", "pac_profile_read", "pac_profile_last_kernel", "pac_version",
            "pac_merge_sizes", "pac_merge_pack", "pac_merge_unpack", "pac_approx_sum_workspace_size",
            "pac_approx_sum"]
