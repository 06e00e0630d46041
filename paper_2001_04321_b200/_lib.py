"""ctypes binding of libntf_b200.so (include/ntf_b200.h).

The library is built in-tree (``paper_2001_04321_b200/libntf_b200.so``) by
``__graft_entry__.build()`` / ``make -C paper_2001_04321_b200/csrc``. There is
no fallback: if the shared object is missing, importing this module fails.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# NTF_B200_LIB: a diagnostics build (e.g. -DNTF_NNLS_PROFILE=1) of the same library
LIB_PATH = os.environ.get("NTF_B200_LIB") or os.path.join(_HERE, "libntf_b200.so")

NTF_OK = 0
NTF_ERR_INVALID_ARGUMENT = 1
NTF_ERR_LOGIC = 2
NTF_ERR_RUNTIME = 3
NTF_ERR_CUDA = 4
NTF_ERR_NCCL = 5
NTF_ERR_UNSUPPORTED = 6

NTF_DTYPE_F64 = 0
NTF_DTYPE_F32 = 1

NTF_RUN_DIMTREE = 1
NTF_RUN_NO_GRAPH = 2
NTF_RUN_GENERIC = 4
NTF_RUN_DIRECT = 8
NTF_RUN_NO_OVERLAP = 16

dptr = C.POINTER(C.c_double)
iptr = C.POINTER(C.c_int)
i64ptr = C.POINTER(C.c_int64)


class InnerStopC(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("rel_change_tol", C.c_double)]


class AoConfigC(C.Structure):
    _fields_ = [("solver", C.c_int), ("inner_stop", InnerStopC), ("max_outer_iters", C.c_int),
                ("max_time_s", C.c_double), ("record_factor_error", C.c_int),
                ("ground_truth", dptr), ("flags", C.c_uint)]


class HerParamsC(C.Structure):
    _fields_ = [("beta0", C.c_double), ("gamma", C.c_double), ("gamma_bar", C.c_double), ("eta", C.c_double)]


class TraceRecordC(C.Structure):
    _fields_ = [("iter", C.c_int), ("has_e", C.c_int), ("has_restarted", C.c_int), ("restarted", C.c_int),
                ("has_beta", C.c_int), ("inner_sweeps", C.c_int), ("time_s", C.c_double), ("f", C.c_double),
                ("e", C.c_double), ("beta", C.c_double)]


class HerIterationInfoC(C.Structure):
    _fields_ = [("iter", C.c_int), ("f_hat", C.c_double), ("restarted", C.c_int), ("beta_used", C.c_double),
                ("factors", dptr), ("hat_factors", dptr)]


OBSERVER = C.CFUNCTYPE(None, C.POINTER(HerIterationInfoC), C.c_void_p)

# name -> (restype, argtypes); every symbol include/ntf_b200.h declares.
SIGNATURES = {
    "ntf_version": (C.c_char_p, []),
    "ntf_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
    "ntf_her_params_default": (None, [C.POINTER(HerParamsC)]),
    "ntf_ao_config_default": (None, [C.POINTER(AoConfigC)]),
    "ntf_her_params_validate": (C.c_int, [C.POINTER(HerParamsC)]),
    "ntf_ao_config_validate": (C.c_int, [C.POINTER(AoConfigC)]),
    "ntf_stream_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "ntf_random_init": (C.c_int, [iptr, C.c_int, C.c_int, C.c_uint64, dptr]),
    "ntf_generate": (C.c_int, [iptr, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_uint64, C.c_int,
                               C.c_void_p, dptr]),
    "ntf_generate_slab": (C.c_int, [iptr, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                    C.c_int64, C.c_int64, C.c_void_p, dptr]),
    "ntf_factor_error": (C.c_int, [dptr, dptr, iptr, C.c_int, C.c_int, dptr]),
    "ntf_ntft_info": (C.c_int, [C.c_char_p, iptr, C.POINTER(C.c_int64)]),
    "ntf_ntft_read": (C.c_int, [C.c_char_p, C.c_int, C.c_int64, C.c_int64, C.c_void_p]),
    "ntf_ntft_write": (C.c_int, [C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int64)]),
    "ntf_tensor_upload_ntft": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "ntf_device_count": (C.c_int, [iptr]),
    "ntf_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "ntf_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "ntf_ctx_create_dist": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(C.c_void_p)]),
    "ntf_ctx_info": (C.c_int, [C.c_void_p, iptr, iptr, iptr]),
    "ntf_ctx_destroy": (C.c_int, [C.c_void_p]),
    "ntf_slab_range": (C.c_int, [C.c_int64, C.c_int, C.c_int, i64ptr, i64ptr]),
    "ntf_tensor_upload": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, i64ptr, C.POINTER(C.c_void_p)]),
    "ntf_tensor_upload_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, i64ptr, C.POINTER(C.c_void_p)]),
    "ntf_tensor_wait": (C.c_int, [C.c_void_p]),
    "ntf_pinned_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "ntf_pinned_free": (C.c_int, [C.c_void_p]),
    "ntf_tensor_upload_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, i64ptr,
                                           C.POINTER(C.c_void_p)]),
    "ntf_tensor_upload_device_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, i64ptr, C.c_void_p,
                                                 C.POINTER(C.c_void_p)]),
    "ntf_tensor_upload_rows": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, i64ptr, C.c_int64, C.c_int64,
                                         C.POINTER(C.c_void_p)]),
    "ntf_tucker_upload": (C.c_int, [C.c_void_p, dptr, C.c_int, i64ptr, dptr, i64ptr, C.POINTER(C.c_void_p)]),
    "ntf_ntfk_info": (C.c_int, [C.c_char_p, iptr, i64ptr, i64ptr]),
    "ntf_ntfk_read": (C.c_int, [C.c_char_p, dptr, dptr]),
    "ntf_ntfk_write": (C.c_int, [C.c_char_p, dptr, dptr, C.c_int, i64ptr, i64ptr]),
    "ntf_tensor_upload_ntfk": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "ntf_tensor_shape": (C.c_int, [C.c_void_p, iptr, i64ptr]),
    "ntf_tensor_norm_sq": (C.c_int, [C.c_void_p, dptr]),
    "ntf_tensor_destroy": (C.c_int, [C.c_void_p]),
    "ntf_mttkrp": (C.c_int, [C.c_void_p, C.c_void_p, dptr, C.c_int, C.c_int, dptr]),
    "ntf_mttkrp_all": (C.c_int, [C.c_void_p, C.c_void_p, dptr, C.c_int, C.c_uint, dptr]),
    "ntf_mttkrp_plan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
    "ntf_objective": (C.c_int, [C.c_void_p, C.c_void_p, dptr, C.c_int, C.c_int, dptr]),
    "ntf_solve_nnls": (C.c_int, [C.c_void_p, C.c_int, dptr, dptr, dptr, C.c_int, C.c_int,
                                 C.POINTER(InnerStopC), dptr, iptr]),
    "ntf_her_run": (C.c_int, [C.c_void_p, C.c_void_p, dptr, C.c_int, C.POINTER(AoConfigC),
                              C.POINTER(HerParamsC), OBSERVER, C.c_void_p, dptr, dptr,
                              C.POINTER(TraceRecordC), C.c_int, iptr]),
    "ntf_ao_run": (C.c_int, [C.c_void_p, C.c_void_p, dptr, C.c_int, C.POINTER(AoConfigC), dptr, dptr,
                             C.POINTER(TraceRecordC), C.c_int, iptr]),
    "ntf_session_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, dptr, C.c_int, C.POINTER(AoConfigC),
                                     C.POINTER(HerParamsC), C.POINTER(C.c_void_p)]),
    "ntf_session_step": (C.c_int, [C.c_void_p, C.c_int]),
    "ntf_session_sync": (C.c_int, [C.c_void_p]),
    "ntf_session_stream": (C.c_void_p, [C.c_void_p]),
    "ntf_session_iterations": (C.c_int, [C.c_void_p, iptr]),
    "ntf_session_factors": (C.c_int, [C.c_void_p, dptr]),
    "ntf_session_trace": (C.c_int, [C.c_void_p, dptr, C.POINTER(TraceRecordC), C.c_int, iptr]),
    "ntf_session_set_kernel_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "ntf_session_kernel_times": (C.c_int, [C.c_void_p, dptr, iptr, iptr]),
    "ntf_session_pass_slots": (C.c_int, [C.c_void_p, iptr, iptr]),
    "ntf_session_destroy": (C.c_int, [C.c_void_p]),
}

_LIB = None


def lib():
    """The loaded CDLL; raises ImportError when the extension is not built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB
