"""ctypes loader for libmxmoe.so (the C ABI of include/mxmoe.h).

Argument marshalling only. If the shared library is missing this raises: there is no
CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmxmoe.so")

MXM_OK, MXM_E_CONFIG, MXM_E_DATA, MXM_E_CUDA, MXM_E_NCCL = 0, 3, 4, 5, 6
# include/mxmoe.h MXM_WS_* (workspace introspection, test-only)
WS_NAMES = ["row_src", "row_w", "row_exp", "inv", "xb", "xqa", "xsa", "xqb", "xsb", "h", "hq", "hs", "o", "v_off",
            "R", "f_max", "xca", "xcb", "hc", "tasks", "meta", "g_max"]


class MxmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"mxmoe status {status}: {msg}")
        self.status = status


class mxm_scheme(C.Structure):
    _fields_ = [("w_bits", C.c_int32), ("a_bits", C.c_int32), ("w_group", C.c_int32), ("a_group", C.c_int32),
                ("symmetric", C.c_int32), ("fmt", C.c_int32)]


class mxm_linear(C.Structure):
    _fields_ = [("scheme", mxm_scheme), ("packed", C.c_void_p)]


class mxm_layer_desc(C.Structure):
    _fields_ = [("n_routed", C.c_int32), ("n_shared", C.c_int32), ("hidden", C.c_int32), ("inter", C.c_int32),
                ("shared_inter", C.c_int32), ("blocks", C.POINTER(mxm_linear))]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_S = C.POINTER(mxm_scheme)

SIGNATURES = {
    "mxm_scheme_check": (C.c_int, [_S, _I64, _I64]),
    "mxm_quant_sizes": (C.c_int, [_S, _I64, _I64, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64)]),
    "mxm_storage_bits_per_weight": (C.c_double, [_S, _I64]),
    "mxm_quantize": (C.c_int, [_S, _P, _I64, _I64, _P, _P, _P, _P, _P]),
    "mxm_pack": (C.c_int, [_S, _P, _P, _P, _I64, _I64, _P, _P]),
    "mxm_dequantize": (C.c_int, [_S, _P, _I64, _I64, _P, _P]),
    "mxm_act_quant": (C.c_int, [_P, _I64, _I64, _I32, _I32, _P, _P, _P, _P]),
    "mxm_route_scratch_bytes": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
    "mxm_route_prep": (C.c_int, [_P, _I64, _I32, _I32, _P, _P, _P, _P, _P, _I64, _P]),
    "mxm_layer_desc_bytes": (C.c_int, [C.POINTER(mxm_layer_desc), C.POINTER(_I64)]),
    "mxm_layer_init": (C.c_int, [C.POINTER(mxm_layer_desc), _P, _I64, _P, C.POINTER(_P)]),
    "mxm_layer_free": (None, [_P]),
    "mxm_workspace_bytes": (C.c_int, [_P, _I64, _I32, C.POINTER(_I64)]),
    "mxm_moe_group_gemm": (C.c_int, [_P, _P, _I64, _I32, _P, _P, _P, _P, _P, _I64, _P]),
    "mxm_poll_device_error": (C.c_int, [_P, _P, _P, C.POINTER(_I32)]),
    "mxm_debug_task_stats": (C.c_int, [_P, _P, _I64, _I32, _P, C.POINTER(_I32), C.POINTER(_I32)]),
    "mxm_layer_profile": (C.c_int, [_P, _I32]),
    "mxm_layer_profile_read": (C.c_int, [_P, _P, _I32, C.POINTER(_I32)]),
    "mxm_kernels_per_call": (C.c_int32, [_P]),
    "mxm_layer_debug_counters": (C.c_int, [_P, _P]),
    "mxm_ep_route": (C.c_int, [_P, _I64, _I32, _I32, _I32, _P, _P, _P, _P]),
    "mxm_ep_pack": (C.c_int, [_P, _I64, _I32, _P, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "mxm_ep_combine": (C.c_int, [_P, _P, _P, _I32, _I64, _I32, _P, _P, _P]),
    "mxm_debug_workspace_layout": (C.c_int, [_P, _I64, _I32, C.POINTER(_I64)]),
    "mxm_debug_acc_bytes": (C.c_int, [_P, _I64, _I32, C.POINTER(_I64)]),
    "mxm_debug_moe_group_gemm_dump": (C.c_int, [_P, _P, _I64, _I32, _P, _P, _P, _P, _P, _I64, _P, _I64, _P]),
    "mxm_profile_scratch_bytes": (C.c_int, [_P, C.POINTER(_I64)]),
    "mxm_profile_tile_costs": (C.c_int, [_P, _P, _I64, _P, _P]),
    "mxm_layer_set_tile_costs": (C.c_int, [_P, _P]),
    "mxm_ep_init": (C.c_int, [_P, _P, _P, _I32, C.POINTER(_P)]),
    "mxm_ep_free": (None, [_P]),
    "mxm_ep_workspace_bytes": (C.c_int, [_P, _I64, _I32, _I64, C.POINTER(_I64)]),
    "mxm_ep_moe_group_gemm": (C.c_int, [_P, _P, _I64, _I32, _P, _P, _P, _P, _P, _I64, _I64, _P]),
    "mxm_ep_poll_device_error": (C.c_int, [_P, _P, _P, C.POINTER(_I32)]),
    "mxm_ep_set_mode": (C.c_int, [_P, _I32]),
    "mxm_hadamard_rotate": (C.c_int, [_P, _P, _I64, _I64, _P, _I32, _P]),
    "mxm_gptq_hessian": (C.c_int, [_P, _I64, _I64, _P, _P]),
    "mxm_gptq_prepare": (C.c_int, [_P, _I64, C.c_double, _P, _P, _P, _P]),
    "mxm_gptq_work_bytes": (C.c_int64, [_I64, _I64]),
    "mxm_gptq_quantize": (C.c_int, [_S, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "mxm_last_error": (C.c_char_p, []),
    "mxm_version": (C.c_char_p, []),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libmxmoe.so and bind every exported symbol of include/mxmoe.h."""
    global _lib
    if _lib is not None:
        return _lib
    # experiment variants built in-tree by build.build_variant (tools/); default: the product library
    path = os.environ.get("MXM_LIB") or path
    if not os.path.exists(path):
        raise MxmError(MXM_E_CUDA, f"{path} not built; run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        if path != LIB_PATH and not hasattr(lib, name):
            continue  # an older experiment variant (tools/variants) may lack newer debug entries
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status != MXM_OK:
        raise MxmError(status, load().mxm_last_error().decode())
