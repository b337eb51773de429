"""ctypes binding of the C-ABI (include/tridpart_b200.h) to the in-tree
``lib/libtridpart_b200.so``. There is no fallback: if the library is missing
or cannot load, importing the package fails loudly."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TPB_LIB overrides the library path (A/B experiments between two builds)
LIB_PATH = os.environ.get("TPB_LIB") or os.path.join(HERE, "lib", "libtridpart_b200.so")

_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_I32 = C.POINTER(C.c_int32)


class TpError(C.Structure):
    _fields_ = [("code", C.c_int32), ("level", C.c_int32), ("row", C.c_int64), ("msg", C.c_char * 256)]


class TpObservation(C.Structure):
    _fields_ = [("n", C.c_int64), ("label", C.c_int32), ("corrected", C.c_int32),
                ("has_corrected", C.c_int32), ("depth_label", C.c_int32), ("streams", C.c_int32),
                ("ntimes", C.c_int32), ("precision", C.c_char * 16), ("device", C.c_char * 48)]


INTERFACE_CB = C.CFUNCTYPE(None, C.c_int64, C.c_int64, _D, _D, _D, _D, C.c_void_p)
_F = C.POINTER(C.c_float)
INTERFACE_CB_F32 = C.CFUNCTYPE(None, C.c_int64, C.c_int64, _F, _F, _F, _F, C.c_void_p)

# tp_status
OK, ZERO_PIVOT, INVALID_SIZE, DEPTH_OUT_OF_RANGE, EMPTY_TRAINING_SET, K_TOO_LARGE = 0, 1, 2, 3, 4, 5
MALFORMED_HEADER, BAD_NUMBER, IO, CUDA, INVALID_ARGUMENT, NCCL = 6, 7, 8, 9, 10, 11

EXPORTS = [
    "tp_abi_version", "tp_ctx_create", "tp_ctx_destroy", "tp_ctx_set_stream", "tp_ctx_set_graphs", "tp_ctx_set_grid",
    "tp_ctx_last_launch_count", "tp_ctx_last_kernels", "tp_solve_partition_f64", "tp_solve_partition_f64_dev",
    "tp_check_device_error", "tp_solve_partition_observe_f64", "tp_thomas_solve_f64",
    "tp_residual_inf_f64_dev", "tp_shard_reduce_f64_dev", "tp_shard_finish_f64_dev",
    "tp_generate_system_f64_dev", "tp_make_plan", "tp_plan_levels", "tp_solve_profile_f64_dev",
    "tp_predict", "tp_fit_knn", "tp_recursion_sizes", "tp_default_model", "tp_obs_read",
    "tp_obs_get", "tp_obs_free", "tp_diag_rcp_ulp", "tp_debug_grid_trace", "tp_solve_partition_f32",
    "tp_solve_partition_f32_dev", "tp_solve_partition_observe_f32", "tp_thomas_solve_f32",
    "tp_residual_inf_f32_dev", "tp_generate_system_f32_dev", "tp_solve_partition_f64_async",
    "tp_solve_partition_f32_async", "tp_shard_mailbox", "tp_ipc_get_handle", "tp_ipc_open_handle",
    "tp_shard_attach", "tp_shard_solve_f64_dev", "tp_shard_prepare_f64_dev",
    "tp_reduce_block_f64", "tp_reduce_block_f32", "tp_generate_system_f64",
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2510_27351_b200/csrc). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    if lib.tp_abi_version() != 2:
        raise ImportError(f"{LIB_PATH}: C-ABI version {lib.tp_abi_version()}, this package needs 2 (rebuild)")
    vp, E = C.c_void_p, C.POINTER(TpError)
    sig = {
        "tp_abi_version": (C.c_int32, []),
        "tp_ctx_create": (C.c_int, [C.c_int32, C.POINTER(vp), E]),
        "tp_ctx_destroy": (None, [vp]),
        "tp_ctx_set_stream": (C.c_int, [vp, vp, E]),
        "tp_ctx_set_graphs": (C.c_int, [vp, C.c_int32, E]),
        "tp_ctx_set_grid": (C.c_int, [vp, C.c_int32, C.c_int64, E]),
        "tp_ctx_last_launch_count": (C.c_int64, [vp]),
        "tp_ctx_last_kernels": (C.c_int64, [vp, C.c_char_p, C.c_int64]),
        "tp_solve_partition_f64": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32, vp, E]),
        "tp_solve_partition_f64_dev": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32, vp,
                                                 vp, E]),
        "tp_check_device_error": (C.c_int, [vp, E]),
        "tp_solve_partition_observe_f64": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32,
                                                     vp, INTERFACE_CB, vp, E]),
        "tp_thomas_solve_f64": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, vp, E]),
        "tp_residual_inf_f64_dev": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, vp, _D, vp, E]),
        "tp_shard_reduce_f64_dev": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32, vp,
                                              vp, E]),
        "tp_shard_finish_f64_dev": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32, vp,
                                              C.c_int32, C.c_int32, vp, vp, E]),
        "tp_generate_system_f64_dev": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                                 C.c_double, vp, vp, vp, vp, vp, E]),
        "tp_make_plan": (C.c_int, [C.c_int64, C.c_int64, _I64, _I64, E]),
        "tp_plan_levels": (C.c_int, [C.c_int64, _I64, C.c_int32, _I64, _I64, _I32, C.c_int32, _I64, E]),
        "tp_solve_profile_f64_dev": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32, vp,
                                               C.POINTER(C.c_float), C.c_char_p, C.c_int32, _I32, E]),
        "tp_predict": (C.c_int, [_I64, _I32, C.c_int64, C.c_int32, C.c_int64, _I32, E]),
        "tp_fit_knn": (C.c_int, [_I64, _I32, C.c_int64, C.c_int32, E]),
        "tp_recursion_sizes": (C.c_int, [C.c_int64, C.c_int32, _I64, _I32, C.c_int64, C.c_int32, _I64,
                                         _I32, E]),
        "tp_default_model": (C.c_int, [C.c_int32, _I64, _I32, C.c_int64, _I64, _I32, E]),
        "tp_obs_read": (C.c_int, [C.c_char_p, C.POINTER(vp), _I64, E]),
        "tp_obs_get": (C.c_int, [vp, C.c_int64, C.POINTER(TpObservation), _I32, _D, E]),
        "tp_obs_free": (None, [vp]),
        "tp_diag_rcp_ulp": (C.c_int, [C.c_int64, C.c_uint64, C.POINTER(C.c_uint64)]),
        "tp_debug_grid_trace": (C.c_int, [C.c_void_p, C.c_int]),
        "tp_solve_partition_f32": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32, vp, E]),
        "tp_solve_partition_f32_dev": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32, vp,
                                                 vp, E]),
        "tp_solve_partition_observe_f32": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32,
                                                     vp, INTERFACE_CB_F32, vp, E]),
        "tp_thomas_solve_f32": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, vp, E]),
        "tp_solve_partition_f64_async": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32, vp,
                                                   vp, E]),
        "tp_solve_partition_f32_async": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32, vp,
                                                   vp, E]),
        "tp_residual_inf_f32_dev": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, vp, _D, vp, E]),
        "tp_reduce_block_f64": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, C.c_int64, C.c_int64, vp, vp, vp,
                                          vp, vp, E]),
        "tp_reduce_block_f32": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, C.c_int64, C.c_int64, vp, vp, vp,
                                          vp, vp, E]),
        "tp_generate_system_f64": (C.c_int, [C.c_int64, C.c_uint64, C.c_double, vp, vp, vp, vp, E]),
        "tp_shard_mailbox": (C.c_int, [vp, C.c_int32, C.POINTER(vp), E]),
        "tp_ipc_get_handle": (C.c_int, [vp, vp, C.POINTER(C.c_uint8), E]),
        "tp_ipc_open_handle": (C.c_int, [vp, C.POINTER(C.c_uint8), C.POINTER(vp), E]),
        "tp_shard_attach": (C.c_int, [vp, C.c_int32, C.c_int32, C.POINTER(vp), E]),
        "tp_shard_solve_f64_dev": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32, vp, vp, E]),
        "tp_shard_prepare_f64_dev": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64, _I64, C.c_int32, vp, vp, E]),
        "tp_generate_system_f32_dev": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                                 C.c_double, vp, vp, vp, vp, vp, E]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
