"""ctypes binding of libsad.so — argument marshalling only, same names as include/sad.h.

Every function raises SadError on a negative return code. The library must be
built in-tree (``python -m paper_0901_2742_b200.build``); there is no fallback.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SAD_LIB_PATH", os.path.join(HERE, "libsad.so"))   # override: A/B experiments

SAD_PROTEIN20, SAD_DNA4 = 0, 1
SAD_F_KEEP_SIM, SAD_F_KERNEL_ALU, SAD_F_KERNEL_TC, SAD_F_TC_INT8, SAD_F_TC_1SM, SAD_F_TC_ALL_LAYERS = 1, 2, 4, 8, 16, 32
SAD_F_RANK_SAMPLES = 64
SAD_F_F1_CUDA_CORES = 128
SAD_F_TILE_SPLIT = 512
SAD_MEM_HOST, SAD_MEM_DEVICE, SAD_MEM_DEVICE_REBASE = 0, 1, 2
ERRORS = {-1: "SAD_E_ARG", -2: "SAD_E_STATE", -3: "SAD_E_SYMBOL", -4: "SAD_E_TOO_SHORT", -5: "SAD_E_TOO_LONG",
          -6: "SAD_E_INSUFFICIENT", -7: "SAD_E_EMPTY", -8: "SAD_E_CAPACITY", -9: "SAD_E_CUDA", -10: "SAD_E_NCCL",
          -11: "SAD_E_OOM", -12: "SAD_E_REPLAN"}
SAD_E_CAPACITY, SAD_E_NCCL, SAD_E_REPLAN = -8, -10, -12

# every symbol include/sad.h declares (checked by tests/test_abi.py)
SYMBOLS = [
    "sad_abi_version", "sad_create", "sad_destroy", "sad_last_error", "sad_error_location", "sad_workspace_size",
    "sad_load", "sad_build_profiles", "sad_operand_size", "sad_ancestor_record_bytes", "sad_rank_local",
    "sad_rank_global", "sad_partition_plan", "sad_exchange_sizes", "sad_pack_plan", "sad_pack", "sad_output_size",
    "sad_output_layout", "sad_finish", "sad_get_local_rank", "sad_get_ancestors", "sad_get_ranks", "sad_get_sorted",
    "sad_get_pivots", "sad_get_bucket", "sad_get_bucket_sizes", "sad_get_similarity", "sad_get_profile_info", "sad_get_stats",
    "sad_reset_stats", "sad_selftest_fixed_point", "sad_get_bucket_view", "sad_get_distance", "sad_exchange_records", "sad_get_distance_f64",
    "sad_upgma_workspace", "sad_upgma", "sad_get_load_report", "sad_nccl_unique_id", "sad_abort", "sad_rank",
    "sad_partition", "sad_output_bound", "sad_graph_account", "sad_exchange_verdict", "sad_key_index_bits",
]


class SadConfig(ctypes.Structure):
    _fields_ = [("alphabet", ctypes.c_int32), ("k", ctypes.c_int32), ("p", ctypes.c_int32),
                ("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("device", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("flags", ctypes.c_uint32)]


class SadError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str = "", location=(-1, -1)):
        self.code = code
        self.name = ERRORS.get(code, str(code))
        self.location = location
        super().__init__(f"{fn}: {self.name}: {msg}")


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_0901_2742_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_size_t
    sig = {
        "sad_abi_version": (u32, []),
        "sad_create": (i32, [ctypes.POINTER(SadConfig), P, ctypes.POINTER(P)]),
        "sad_nccl_unique_id": (i32, [P]),
        "sad_abort": (i32, [P]),
        "sad_rank": (i32, [P, P, sz]),
        "sad_partition": (i32, [P, P, sz, P]),
        "sad_output_bound": (i32, [P, i64, ctypes.POINTER(sz)]),
        "sad_graph_account": (i32, [P]),
        "sad_exchange_verdict": (i32, [i32, i32, P, P, P, P]),
        "sad_key_index_bits": (i32, [P]),
        "sad_destroy": (None, [P]),
        "sad_last_error": (ctypes.c_char_p, [P]),
        "sad_error_location": (i32, [P, P, P]),
        "sad_workspace_size": (i32, [P, i64, i64, ctypes.POINTER(sz)]),
        "sad_load": (i32, [P, P, P, i64, i64, i64, i64, i32, P, sz]),
        "sad_build_profiles": (i32, [P]),
        "sad_operand_size": (i32, [P, ctypes.POINTER(sz)]),
        "sad_ancestor_record_bytes": (sz, [P]),
        "sad_rank_local": (i32, [P, P, sz, P]),
        "sad_rank_global": (i32, [P, P, P]),
        "sad_partition_plan": (i32, [P, P, P]),
        "sad_exchange_sizes": (i32, [i32, i32, i32, P, P, P, P, P]),
        "sad_pack_plan": (i32, [i32, i32, i32, P, P]),
        "sad_pack": (i32, [P, P, P, P]),
        "sad_output_size": (i32, [P, P, ctypes.POINTER(sz)]),
        "sad_output_layout": (i32, [P, P, P]),
        "sad_finish": (i32, [P, P, P, P, P, sz, P]),
        "sad_get_local_rank": (i32, [P, i32, P, i64]),
        "sad_get_ancestors": (i32, [P, P, P]),
        "sad_get_ranks": (i32, [P, i32, P, P, P, i64]),
        "sad_get_sorted": (i32, [P, i32, P, i64]),
        "sad_get_pivots": (i32, [P, P]),
        "sad_get_bucket": (i32, [P, i32, P, P, P, P, i64, i64, P, P]),
        "sad_get_bucket_sizes": (i32, [P, P]),
        "sad_get_load_report": (i32, [P, P]),
        "sad_get_similarity": (i32, [P, i32, P, i64]),
        "sad_get_profile_info": (i32, [P, P, P, P]),
        "sad_get_stats": (i32, [P, P, P]),
        "sad_reset_stats": (i32, [P]),
        "sad_selftest_fixed_point": (i32, [P, i32, P]),
        "sad_get_bucket_view": (i32, [P, i32, P, P, P, P]),
        "sad_get_distance": (i32, [P, i32, P, i64]),
        "sad_exchange_records": (i32, [P]),
        "sad_get_distance_f64": (i32, [P, i32, P, i64]),
        "sad_upgma_workspace": (sz, [i64]),
        "sad_upgma": (i32, [P, i64, P, P, P, P, sz, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int, fn: str, ctx=None):
    if rc < 0:
        msg, loc = "", (-1, -1)
        if ctx:
            m = lib().sad_last_error(ctx)
            msg = m.decode() if m else ""
            a, b = ctypes.c_int64(-1), ctypes.c_int64(-1)
            lib().sad_error_location(ctx, ctypes.byref(a), ctypes.byref(b))
            loc = (a.value, b.value)
        raise SadError(rc, fn, msg, loc)
    return rc


def call(name: str, *args, ctx=None):
    """Call a sad_* entry point; raise SadError on a negative result."""
    rc = getattr(lib(), name)(*args)
    if isinstance(rc, int):
        check(rc, name, ctx)
    return rc
