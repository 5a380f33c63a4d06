"""ctypes binding of include/treeattn_b200.h (libtreeattn_b200.so, built in-tree).

Importing this module loads the native library and fails loudly when it is
missing -- there is no Python/CPU fallback for the attention path.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TREEATTN_B200_LIB") or os.path.join(_PKG, "libtreeattn_b200.so")   # env: A/B experiments

TA_OK = 0
TA_ERR_INVALID_ARGUMENT = 1
TA_ERR_OUT_OF_RANGE = 2
TA_ERR_LOGIC = 3
TA_ERR_CUDA = 4
TA_ERR_NO_DEVICE = 5
TA_ERR_OUT_OF_MEMORY = 6
TA_F32 = 0
TA_BF16 = 1

# Every symbol include/treeattn_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = [
    "ta_last_error", "ta_abi_version", "ta_ctx_create", "ta_ctx_destroy", "ta_set_option",
    "ta_tree_new", "ta_tree_restore", "ta_tree_branch", "ta_tree_prune", "ta_tree_append",
    "ta_tree_leaves", "ta_tree_get_info", "ta_tree_snapshot", "ta_pool_stats", "ta_pool_token_ref",
    "ta_kv_write", "ta_plan_flatten", "ta_plan_json", "ta_prepare", "ta_attend", "ta_attend_host", "ta_attend_host_async", "ta_attend_host_wait",
    "ta_io_stats_get", "ta_launches_per_attend", "ta_schedule_get",
    "ta_tree_append_leaves", "ta_kv_append", "ta_kv_append_rows", "ta_graph_epoch",
    "ta_io_measured", "ta_io_analytical", "ta_lse_merge", "ta_fast_prepares",
]

TA_STRATEGY = {"q-guided": 0, "node": 1, "node-chunk": 2, "flatten": 3}
TA_ALG = {"naive": 0, "flash-decoding": 1, "radix": 2, "tree-attn-medusa": 3, "tree-attn-specinfer": 4,
          "node": 5, "node-chunk": 6, "flatten": 7}


class CostParams(C.Structure):
    _fields_ = [("d_head", C.c_int), ("n_heads", C.c_int), ("n_layers", C.c_int), ("dtype_bytes", C.c_int)]


class IoReport(C.Structure):
    _fields_ = [("kv_bytes", C.c_uint64), ("q_bytes", C.c_uint64), ("mask_bytes", C.c_uint64),
                ("partial_bytes", C.c_uint64)]


class TreeAttnError(Exception):
    code = -1


class InvalidArgument(TreeAttnError, ValueError):
    code = TA_ERR_INVALID_ARGUMENT


class OutOfRange(TreeAttnError, IndexError):
    code = TA_ERR_OUT_OF_RANGE


class LogicError(TreeAttnError, RuntimeError):
    code = TA_ERR_LOGIC


class CudaError(TreeAttnError, RuntimeError):
    code = TA_ERR_CUDA


class NoDevice(TreeAttnError, RuntimeError):
    code = TA_ERR_NO_DEVICE


class OutOfMemory(TreeAttnError, MemoryError):
    code = TA_ERR_OUT_OF_MEMORY


_ERRS = {c.code: c for c in (InvalidArgument, OutOfRange, LogicError, CudaError, NoDevice, OutOfMemory)}


class Shape(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("n_q_heads", C.c_int), ("n_kv_heads", C.c_int),
                ("d_head", C.c_int), ("kv_dtype", C.c_int), ("out_dtype", C.c_int),
                ("page_tokens", C.c_int), ("kv_head_begin", C.c_int), ("n_local_kv_heads", C.c_int),
                ("max_pages", C.c_int64)]


class TreeInfo(C.Structure):
    _fields_ = [("root", C.c_int32), ("node_count", C.c_int32), ("n_leaves", C.c_int32),
                ("next_id", C.c_int32), ("total_tokens", C.c_int64), ("path_tokens_sum", C.c_int64)]


class PlanView(C.Structure):
    _fields_ = [("block_size", C.c_int), ("n_groups", C.c_int),
                ("seg_begin", C.POINTER(C.c_int32)), ("q_begin", C.POINTER(C.c_int32)),
                ("seg_node", C.POINTER(C.c_int32)), ("seg_offset", C.POINTER(C.c_int64)),
                ("seg_len", C.POINTER(C.c_int64)), ("seg_mask", C.POINTER(C.c_uint64)),
                ("queries", C.POINTER(C.c_int32))]


class IoStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "n_chunks", "n_groups", "n_units", "n_units_mma", "n_partials", "kv_bytes", "kv_bytes_loaded",
        "q_bytes", "out_bytes", "partial_bytes", "meta_bytes", "flops", "host_plan_ns", "host_schedule_ns",
        "host_upload_ns")]


class ScheduleView(C.Structure):
    _fields_ = [("n_ctas", C.c_int32), ("cta_begin", C.POINTER(C.c_int32)),
                ("n_items", C.c_int32), ("items", C.POINTER(C.c_int32)),
                ("n_tiles", C.c_int32), ("tiles", C.POINTER(C.c_int32)),
                ("n_grp", C.c_int32), ("grp_row", C.POINTER(C.c_int32)), ("grp_info", C.POINTER(C.c_uint32)),
                ("n_slot_leaf", C.c_int32), ("slot_leaf", C.POINTER(C.c_int32)),
                ("n_slot_out", C.c_int32), ("slot_out", C.POINTER(C.c_int32)),
                ("n_partials", C.c_int32), ("part_merge", C.POINTER(C.c_int32)),
                ("n_merge", C.c_int32), ("merge_leaf", C.POINTER(C.c_int32)),
                ("merge_head", C.POINTER(C.c_int32)), ("merge_begin", C.POINTER(C.c_int32)),
                ("merge_parts", C.POINTER(C.c_int32)),
                ("n_empty", C.c_int32), ("empty", C.POINTER(C.c_int32)),
                ("n_lanes", C.c_int32), ("use_mma", C.c_int32), ("fused_merge", C.c_int32),
                ("cta_pub_begin", C.POINTER(C.c_int32)), ("cta_pub", C.POINTER(C.c_int32)),
                ("cta_own_begin", C.POINTER(C.c_int32)), ("cta_own", C.POINTER(C.c_int32))]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2404_00242_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    pi32, pi64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
    sig = {
        "ta_last_error": (C.c_char_p, []),
        "ta_abi_version": (C.c_int, []),
        "ta_ctx_create": (C.c_int, [C.c_int, C.POINTER(Shape), C.POINTER(vp)]),
        "ta_ctx_destroy": (C.c_int, [vp]),
        "ta_set_option": (C.c_int, [vp, C.c_char_p, i64]),
        "ta_tree_new": (C.c_int, [vp, i64, pi32]),
        "ta_tree_restore": (C.c_int, [vp, i32, C.c_int, pi32, pi32, pi64]),
        "ta_tree_branch": (C.c_int, [vp, i32, C.c_int, pi64, pi32]),
        "ta_tree_prune": (C.c_int, [vp, i32]),
        "ta_tree_append": (C.c_int, [vp, i32, i64]),
        "ta_tree_leaves": (C.c_int, [vp, pi32, C.c_int, C.POINTER(C.c_int)]),
        "ta_tree_get_info": (C.c_int, [vp, C.POINTER(TreeInfo)]),
        "ta_tree_snapshot": (C.c_int, [vp, pi32, pi32, pi64, C.c_int, C.POINTER(C.c_int)]),
        "ta_pool_stats": (C.c_int, [vp, pi64, pi64, pi64]),
        "ta_pool_token_ref": (C.c_int, [vp, i32, i64, pi32, pi32]),
        "ta_kv_write": (C.c_int, [vp, C.c_int, i32, i64, i64, vp, vp, C.c_int, vp]),
        "ta_plan_flatten": (C.c_int, [vp, C.c_int, C.POINTER(PlanView)]),
        "ta_plan_json": (C.c_int, [vp, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
        "ta_prepare": (C.c_int, [vp, C.c_int, vp]),
        "ta_attend": (C.c_int, [vp, C.c_int, vp, vp, vp, vp]),
        "ta_attend_host": (C.c_int, [vp, C.c_int, vp, vp, vp]),
        "ta_attend_host_async": (C.c_int, [vp, C.c_int, vp, vp, vp]),
        "ta_attend_host_wait": (C.c_int, [vp]),
        "ta_io_stats_get": (C.c_int, [vp, C.POINTER(IoStats)]),
        "ta_launches_per_attend": (C.c_int, [vp]),
        "ta_schedule_get": (C.c_int, [vp, C.c_int, C.POINTER(ScheduleView)]),
        "ta_tree_append_leaves": (C.c_int, [vp, C.c_int, pi32, pi64]),
        "ta_kv_append": (C.c_int, [vp, C.c_int, vp, vp, vp]),
        "ta_kv_append_rows": (i64, [vp]),
        "ta_graph_epoch": (i64, [vp]),
        "ta_fast_prepares": (i64, [vp]),
        "ta_io_measured": (C.c_int, [vp, C.c_int, C.POINTER(CostParams), C.POINTER(IoReport)]),
        "ta_io_analytical": (C.c_int, [vp, C.c_int, C.POINTER(CostParams), C.c_int, C.POINTER(IoReport)]),
        "ta_lse_merge": (C.c_int, [vp, vp, C.c_int, i64, C.c_int, vp, C.c_int, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int, what: str = ""):
    if rc == TA_OK:
        return
    msg = lib().ta_last_error().decode()
    raise _ERRS.get(rc, TreeAttnError)(f"{what}: {msg}" if what else msg)
