"""ctypes loader for libthemis.so (the C ABI in include/themis.h).

Argument marshalling only: every step of the hot path runs in libthemis.
Fails loudly if the library is missing — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libthemis.so")

MAX_DIMS = 8
MAX_GPUS = 8
MAX_CHUNKS = 1024
IPC_HANDLE_BYTES = 64

STATUS = {0: "THEMIS_OK", 1: "THEMIS_ERR_INVALID_ARG", 2: "THEMIS_ERR_ALIGNMENT", 3: "THEMIS_ERR_UNSUPPORTED_DTYPE",
          4: "THEMIS_ERR_OVERFLOW", 5: "THEMIS_ERR_NOT_REGISTERED", 6: "THEMIS_ERR_PLAN_MISMATCH",
          7: "THEMIS_ERR_CUDA", 8: "THEMIS_ERR_TIMEOUT"}


class ThemisError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Topology_t(C.Structure):
    _fields_ = [("ndims", C.c_int32), ("size", C.c_int32 * MAX_DIMS), ("bw_mbps", C.c_uint32 * MAX_DIMS),
                ("step_latency_ns", C.c_uint32 * MAX_DIMS), ("kind", C.c_int32 * MAX_DIMS)]


class PlanReq_t(C.Structure):
    _fields_ = [("coll", C.c_int32), ("policy", C.c_int32), ("intra", C.c_int32), ("n_chunks", C.c_int32),
                ("bytes", C.c_uint64), ("threshold_div", C.c_int32), ("charge_latency", C.c_int32),
                ("concurrency", C.c_int32), ("reserved", C.c_int32), ("chunk_release_ns", C.c_uint64)]


class PlanInfo_t(C.Structure):
    _fields_ = [("ndims", C.c_int32), ("n_chunks", C.c_int32), ("n_ranks", C.c_int32), ("n_stages", C.c_int32),
                ("n_greedy", C.c_int32), ("coll", C.c_int32), ("policy", C.c_int32), ("intra", C.c_int32),
                ("time_scale", C.c_uint64), ("byte_scale", C.c_uint64), ("makespan", C.c_uint64),
                ("busy", C.c_uint64 * MAX_DIMS), ("idle", C.c_uint64 * MAX_DIMS),
                ("dim_volume", C.c_uint64 * MAX_DIMS), ("final_load", C.c_uint64 * MAX_DIMS),
                ("hash", C.c_uint64), ("util_num", C.c_uint64), ("util_den", C.c_uint64),
                ("util_exact", C.c_int32), ("reserved_info", C.c_int32)]


_P = C.c_void_p
_ST = C.c_int
SIGNATURES = {
    "themis_plan": (_ST, [C.POINTER(Topology_t), C.POINTER(PlanReq_t), C.POINTER(_P)]),
    "themis_plan_custom": (_ST, [C.POINTER(Topology_t), C.POINTER(PlanReq_t), _P, _P, C.POINTER(_P)]),
    "themis_plan_info": (_ST, [_P, C.POINTER(PlanInfo_t)]),
    "themis_plan_orders": (_ST, [_P, _P, _P]),
    "themis_plan_dim_ops": (_ST, [_P, _P, _P]),
    "themis_plan_times": (_ST, [_P, _P, _P]),
    "themis_plan_servers": (_ST, [_P, _P]),
    "themis_plan_free": (None, [_P]),
    "themis_heap_layout": (_ST, [C.c_int32, C.c_int32, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint64)]),
    "themis_heap_alloc": (_ST, [C.c_uint64, C.POINTER(_P)]),
    "themis_heap_free": (_ST, [_P]),
    "themis_heap_export": (_ST, [_P, _P]),
    "themis_heap_import": (_ST, [_P, C.POINTER(_P)]),
    "themis_heap_close": (_ST, [_P]),
    "themis_comm_create": (_ST, [C.c_int32, C.c_int32, C.POINTER(Topology_t), C.POINTER(_P), C.c_uint64, C.c_uint64,
                                 C.POINTER(_P)]),
    "themis_comm_free": (None, [_P]),
    "themis_comm_status": (_ST, [_P]),
    "themis_comm_set_engine": (_ST, [_P, C.c_int32]),
    "themis_comm_set_pacing": (_ST, [_P, C.c_int32]),
    "themis_comm_set_stages": (_ST, [_P, C.c_int32]),
    "themis_comm_set_stage_bytes": (_ST, [_P, C.c_int32]),
    "themis_comm_set_min_cta_bytes": (_ST, [_P, C.c_uint64]),
    "themis_comm_set_window_rotation": (_ST, [_P, C.c_int32]),
    "themis_comm_set_lookahead": (_ST, [_P, C.c_int32]),
    "themis_comm_set_push": (_ST, [_P, C.c_int32]),
    "themis_comm_set_ll": (_ST, [_P, C.c_uint64, C.c_uint64]),
    "themis_plan_bound_ll": (_ST, [_P, C.POINTER(C.c_int32)]),
    "themis_comm_set_multicast": (_ST, [_P, _P]),
    "themis_comm_set_timeout": (_ST, [_P, C.c_uint64]),
    "themis_comm_enable_trace": (_ST, [_P, C.c_int32]),
    "themis_trace_fetch": (_ST, [_P, _P, C.c_size_t]),
    "themis_trace_fetch_detail": (_ST, [_P, _P, C.c_size_t]),
    "themis_default_ctas": (_ST, [C.POINTER(Topology_t), C.c_int32, _P]),
    "themis_plan_bind": (_ST, [_P, _P, _P]),
    "themis_plan_bound_ctas": (_ST, [_P, _P]),
    "themis_plan_bound_nvls": (_ST, [_P, C.POINTER(C.c_int32)]),
    "themis_debug_fake_peer_gpu": (_ST, [_P, C.c_int32, C.c_uint64, C.c_int32]),
    "themis_plan_launch_hash": (_ST, [_P, C.c_uint64, C.c_int32, C.POINTER(C.c_uint64)]),
    "themis_allreduce": (_ST, [_P, C.c_uint64, C.c_int32, _P, _P]),
    "themis_reduce_scatter": (_ST, [_P, C.c_uint64, C.c_int32, _P, _P]),
    "themis_all_gather": (_ST, [_P, C.c_uint64, C.c_int32, _P, _P]),
    "themis_allreduce_host": (_ST, [_P, _P, _P, C.c_uint64, C.c_int32, _P, _P]),
    "themis_launches_per_call": (C.c_int32, []),
    "themis_last_error": (C.c_char_p, []),
    "themis_version": (C.c_char_p, []),
}

_lib = None


def lib():
    """Load libthemis.so (built in-tree by paper_2110_04478_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2110_04478_b200.build` "
                              "(or __graft_entry__.build()); there is no fallback implementation")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise ThemisError(status, lib().themis_last_error().decode())
