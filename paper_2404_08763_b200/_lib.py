"""ctypes loader for libcats.so -- declares every symbol of include/cats.h. No fallback: if the
library is missing the import fails loudly (there is no CPU path)."""
from __future__ import annotations

import ctypes
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libcats.so")

CATS_F32, CATS_BF16 = 0, 1
CALIB_MAX_BINS = 32768
STATUS = ["CATS_OK", "CATS_E_NULL", "CATS_E_SHAPE", "CATS_E_DTYPE", "CATS_E_ALIGN", "CATS_E_SPARSITY",
          "CATS_E_EMPTY", "CATS_E_NONFINITE", "CATS_E_THRESHOLD", "CATS_E_BATCH", "CATS_E_WORKSPACE",
          "CATS_E_CUDA", "CATS_E_UNSUPPORTED"]


class CalibInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("rank_r", ctypes.c_uint64), ("count_lt", ctypes.c_uint64),
                ("count_le", ctypes.c_uint64), ("t_bits", ctypes.c_uint32), ("passes", ctypes.c_uint32)]


class CalibWindow(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_uint32), ("hi", ctypes.c_uint32), ("shift", ctypes.c_uint32),
                ("nbins", ctypes.c_uint32), ("sample_stride", ctypes.c_uint64)]


class PlanOptions(ctypes.Structure):
    """cats_mlp_plan_options_t (include/cats.h)."""
    _fields_ = [("size", ctypes.c_uint32), ("path", ctypes.c_int32), ("compaction", ctypes.c_int32),
                ("trace", ctypes.c_int32), ("rows_per_tile", ctypes.c_int32), ("max_stages", ctypes.c_int32),
                ("lazy_tail", ctypes.c_int32), ("min_tiles", ctypes.c_int32), ("eager", ctypes.c_int32),
                ("l2_prefetch", ctypes.c_int32),
                ("xs_cols", ctypes.c_int32), ("xs_ranges", ctypes.c_int32),
                ("xs_mma", ctypes.c_int32), ("xs_no_shrink", ctypes.c_int32)]


CATS_PATH_AUTO, CATS_PATH_FUSED, CATS_PATH_SPLIT = 0, 1, 2
CATS_COMPACT_BALLOT, CATS_COMPACT_PREDICATED, CATS_COMPACT_ATOMIC = 0, 1, 2


class PlanInfo(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int), ("m", ctypes.c_int), ("max_batch", ctypes.c_int), ("w_dtype", ctypes.c_int),
                ("device", ctypes.c_int), ("num_sms", ctypes.c_int), ("grid", ctypes.c_int),
                ("threads", ctypes.c_int), ("rows_per_tile", ctypes.c_int), ("stages", ctypes.c_int),
                ("smem", ctypes.c_size_t), ("workspace_bytes", ctypes.c_size_t)]


_lock = threading.Lock()
_lib = None

P, I, U64, SZ, D, F = (ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_double,
                       ctypes.c_float)
_SIGS = {
    "cats_status_string": (ctypes.c_char_p, [I]),
    "cats_last_cuda_error": (ctypes.c_char_p, []),
    "cats_version": (I, []),
    "cats_calib_rank": (I, [D, U64, P]),
    "cats_calibrate_workspace_bytes": (I, [U64, I, P]),
    "cats_calibrate_threshold": (I, [P, U64, I, D, P, SZ, P, P, P]),
    "cats_calib_window_init": (I, [U64, I, P]),
    "cats_calib_hist": (I, [P, U64, I, P, P, P, P]),
    "cats_calib_step": (I, [P, P, U64, I, D, P, P, P, P, P]),
    "cats_mlp_plan_create": (I, [I, I, I, I, I, I, P]),
    "cats_mlp_plan_options_init": (I, [P]),
    "cats_mlp_plan_create_ex": (I, [I, I, I, I, I, I, P, P]),
    "cats_xsparse_plan_create_ex": (I, [I, I, I, I, I, I, P, P]),
    "cats_mlp_plan_destroy": (None, [P]),
    "cats_mlp_plan_info": (I, [P, P]),
    "cats_mlp_workspace_bytes": (I, [P, P]),
    "cats_mlp_workspace_init": (I, [P, P, SZ, P]),
    "cats_mlp_decode": (I, [P, P, I, P, P, P, F, P, P, SZ, P]),
    "cats_mlp_decode_profiled": (I, [P, P, I, P, P, P, F, P, P, SZ, P, P]),
    "cats_mlp_dense": (I, [P, P, I, P, P, P, P, P, SZ, P]),
    "cats_mlp_decode_host": (I, [P, P, I, P, P, P, F, P, P, SZ, P]),
    "cats_mlp_host_call_create": (I, [P, P, I, P, P, P, F, P, P, SZ, P, P]),
    "cats_mlp_host_call_run": (I, [P]),
    "cats_mlp_host_call_destroy": (None, [P]),
    "cats_mlp_gate_act": (I, [P, P, I, P, P, P, SZ, P]),
    "cats_mlp_last_active": (I, [P, P, I, P, P, P, P, P]),
    "cats_mlp_trace_info": (I, [P, P, P]),
    "cats_mlp_kernels_per_call": (I, [P, I, P]),
    "cats_xsparse_plan_create": (I, [I, I, I, I, I, I, P]),
    "cats_xsparse_gemv": (I, [P, P, I, P, F, P, P, SZ, P]),
    "cats_tp_buffer_bytes": (I, [I, U64, P]),
    "cats_tp_buffer_alloc": (I, [SZ, I, P]),
    "cats_tp_buffer_free": (I, [P]),
    "cats_ipc_handle_get": (I, [P, P]),
    "cats_ipc_handle_open": (I, [P, I, P]),
    "cats_ipc_handle_close": (I, [P]),
    "cats_tp_comm_create": (I, [I, I, U64, P, I, P]),
    "cats_tp_comm_destroy": (None, [P]),
    "cats_tp_allreduce": (I, [P, P, P, U64, P]),
    "cats_tp_allreduce_emulated": (I, [P, I, P, P, U64, P]),
}


def load() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2404_08763_b200.build` "
                                  "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols():
    return list(_SIGS)
