"""ctypes binding of libspmvk.so (the C-ABI declared in include/spmvk.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no CPU fallback: if the library is missing this module raises on
first use, and every compute entry point returns SPMVK_ECUDA without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspmvk.so")

SPMVK_OK, SPMVK_EINVAL, SPMVK_ERANGE, SPMVK_ECUDA, SPMVK_ENCCL, SPMVK_ENOMEM, SPMVK_EPARSE = \
    range(7)
F32, F64 = 4, 8

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p
u64 = C.c_uint64
i64 = C.c_int64
cint = C.c_int


class RgcsrInfo(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "num_rows", "num_cols", "group_size", "num_groups", "slots", "nnz",
        "artificial_zeros", "bytes_single", "bytes_double")] + [("precision", C.c_int),
                                                                ("ellpack", C.c_int)]


class HybridInfo(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "num_rows", "num_cols", "ell_width", "ell_slots", "coo_nnz", "nnz", "fill_nnz",
        "artificial_zeros", "bytes_single", "bytes_double")] + [("precision", C.c_int),
                                                                ("ellpack", C.c_int)]


# name -> (restype, argtypes); every symbol include/spmvk.h declares.
SIGNATURES = {
    "spmvk_last_error": (C.c_char_p, []),
    "spmvk_abi_version": (cint, []),
    "spmvk_init": (cint, [cint]),
    "spmvk_empty_cache": (cint, [cint]),
    "spmvk_host_alloc": (cint, [u64, C.POINTER(vp)]),
    "spmvk_host_free": (cint, [vp]),
    "spmvk_csr_upload": (cint, [u64, u64, u64, vp, vp, vp, cint, vp, C.POINTER(vp)]),
    "spmvk_csr_upload_device": (cint, [u64, u64, u64, vp, vp, vp, cint, vp, C.POINTER(vp)]),
    "spmvk_csr_stencil": (cint, [cint, u64, vp, C.POINTER(vp)]),
    "spmvk_csr_shape": (cint, [vp, u64p, u64p, u64p, C.POINTER(cint)]),
    "spmvk_csr_download": (cint, [vp, vp, vp, vp]),
    "spmvk_csr_row_length_range": (cint, [vp, u64p]),
    "spmvk_csr_column_range": (cint, [vp, u64, u64, u64p]),
    "spmvk_mm_parse": (cint, [C.c_char_p, u64, cint, cint, vp, C.POINTER(vp), u64p]),
    "spmvk_mm_load": (cint, [C.c_char_p, cint, cint, vp, C.POINTER(vp), u64p]),
    "spmvk_mm_write": (cint, [vp, cint, vp, u64, u64p]),
    "spmvk_mm_save": (cint, [vp, C.c_char_p, cint]),
    "spmvk_csr_descending_permutation": (cint, [vp, vp]),
    "spmvk_csr_permute": (cint, [vp, vp, u64, cint, vp, C.POINTER(vp)]),
    "spmvk_permute_vector_f64": (cint, [vp, u64, vp, vp, cint, vp]),
    "spmvk_permute_vector_f32": (cint, [vp, u64, vp, vp, cint, vp]),
    "spmvk_csr_permute_rows_descending": (cint, [vp, vp, C.POINTER(vp), vp]),
    "spmvk_csr_spmv_f64": (cint, [vp, vp, u64, vp, u64, vp]),
    "spmvk_csr_spmv_f32": (cint, [vp, vp, u64, vp, u64, vp]),
    "spmvk_csr_destroy": (None, [vp]),
    "spmvk_rgcsr_build": (cint, [vp, u64, cint, vp, C.POINTER(vp)]),
    "spmvk_rgcsr_build_rows": (cint, [vp, u64, u64, u64, cint, vp, C.POINTER(vp)]),
    "spmvk_rgcsr_get_info": (cint, [vp, C.POINTER(RgcsrInfo)]),
    "spmvk_rgcsr_download": (cint, [vp, vp, vp, vp, vp]),
    "spmvk_rgcsr_to_csr": (cint, [vp, vp, C.POINTER(vp)]),
    "spmvk_hybrid_to_csr": (cint, [vp, vp, C.POINTER(vp)]),
    "spmvk_rgcsr_spmv_f64": (cint, [vp, vp, u64, vp, u64, vp]),
    "spmvk_rgcsr_spmv_f32": (cint, [vp, vp, u64, vp, u64, vp]),
    "spmvk_rgcsr_spmv_scaled_f64": (cint, [vp, vp, u64, vp, u64, vp, C.c_double, vp]),
    "spmvk_rgcsr_spmv_host_f64": (cint, [vp, vp, u64, vp, u64, u64p]),
    "spmvk_rgcsr_spmv_host_f32": (cint, [vp, vp, u64, vp, u64, u64p]),
    "spmvk_rgcsr_destroy": (None, [vp]),
    "spmvk_set_rgcsr_kernel": (cint, [C.c_char_p]),
    "spmvk_set_hybrid_kernel": (cint, [C.c_char_p]),
    "spmvk_stream_persist_x": (cint, [vp, vp, u64, C.c_double, u64p]),
    "spmvk_set_long_row_cut": (cint, [C.c_uint32]),
    "spmvk_set_long_fused": (cint, [cint]),
    "spmvk_csr_choose_ell_width": (cint, [vp, u64p]),
    "spmvk_choose_ell_width": (u64, [vp, u64]),
    "spmvk_hybrid_split_cost": (u64, [vp, u64, u64]),
    "spmvk_hybrid_build": (cint, [vp, i64, cint, vp, C.POINTER(vp)]),
    "spmvk_hybrid_get_info": (cint, [vp, C.POINTER(HybridInfo)]),
    "spmvk_hybrid_download": (cint, [vp, vp, vp, vp, vp, vp]),
    "spmvk_hybrid_spmv_f64": (cint, [vp, vp, u64, vp, u64, vp]),
    "spmvk_hybrid_spmv_f32": (cint, [vp, vp, u64, vp, u64, vp]),
    "spmvk_hybrid_spmv_host_f64": (cint, [vp, vp, u64, vp, u64]),
    "spmvk_hybrid_spmv_host_f32": (cint, [vp, vp, u64, vp, u64]),
    "spmvk_hybrid_destroy": (None, [vp]),
    "spmvk_cg_solve_f64": (cint, [vp, vp, vp, u64, C.c_double, u64, u64, u64p,
                                  C.POINTER(C.c_double), vp]),
    "spmvk_dot_f64": (cint, [vp, vp, u64, vp, vp]),
    "spmvk_rgcsr_spmv_dot_f64": (cint, [vp, vp, u64, vp, u64, u64, vp, vp]),
    "spmvk_cg_update_f64": (cint, [u64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "spmvk_cg_direction_f64": (cint, [u64, vp, vp, vp, vp, vp]),
    "spmvk_ellpack_build": (cint, [vp, u64, cint, vp, C.POINTER(vp)]),
    "spmvk_hybrid_spmv_ell_f64": (cint, [vp, vp, u64, vp, u64, vp]),
    "spmvk_hybrid_spmv_ell_f32": (cint, [vp, vp, u64, vp, u64, vp]),
    "spmvk_hybrid_spmv_coo_f64": (cint, [vp, vp, u64, vp, u64, vp]),
    "spmvk_hybrid_spmv_coo_f32": (cint, [vp, vp, u64, vp, u64, vp]),
    "spmvk_hybrid_spmv_ell_host_f64": (cint, [vp, vp, u64, vp, u64]),
    "spmvk_hybrid_spmv_ell_host_f32": (cint, [vp, vp, u64, vp, u64]),
    "spmvk_hybrid_spmv_coo_host_f64": (cint, [vp, vp, u64, vp, u64]),
    "spmvk_hybrid_spmv_coo_host_f32": (cint, [vp, vp, u64, vp, u64]),
    "spmvk_window_create": (cint, [u64, cint, C.POINTER(vp)]),
    "spmvk_window_ipc_handle": (cint, [vp, vp]),
    "spmvk_window_x": (cint, [vp, cint, C.POINTER(vp)]),
    "spmvk_window_destroy": (None, [vp]),
    "spmvk_dist_open": (cint, [vp, cint, cint, vp, C.POINTER(vp)]),
    "spmvk_dist_open_local": (cint, [C.POINTER(vp), cint, cint, C.POINTER(vp)]),
    "spmvk_dist_set_rows": (cint, [vp, u64, u64, vp]),
    "spmvk_dist_step_f64": (cint, [vp, vp, C.c_double, vp, cint, vp]),
    "spmvk_dist_step_f32": (cint, [vp, vp, C.c_float, vp, cint, vp]),
    "spmvk_dist_cg_direction_f64": (cint, [vp, vp, vp, vp, C.c_int, vp]),
    "spmvk_dist_current": (cint, [vp, C.POINTER(cint)]),
    "spmvk_rgcsr_spmv_scaled_f32": (cint, [vp, vp, u64, vp, u64, vp, C.c_float, vp]),
    "spmvk_plan_slabs": (cint, [u64, u64, cint, u64p, u64p]),
    "spmvk_plan_slabs_weighted": (cint, [vp, u64, u64, cint, u64p]),
    "spmvk_plan_receive": (cint, [cint, u64p, u64p, cint, u64p]),
    "spmvk_plan_halo": (cint, [cint, cint, u64p, u64p, u64p, C.POINTER(cint), u64p,
                                C.POINTER(cint)]),
    "spmvk_nccl_version": (cint, [C.POINTER(cint)]),
    "spmvk_nccl_unique_id": (cint, [vp]),
    "spmvk_comm_init_rank": (cint, [vp, cint, cint, cint, C.POINTER(vp)]),
    "spmvk_comm_init_all": (cint, [cint, vp, vp]),
    "spmvk_comm_info": (cint, [vp, C.POINTER(cint), C.POINTER(cint), C.POINTER(cint)]),
    "spmvk_comm_destroy": (None, [vp]),
    "spmvk_nccl_group_start": (cint, []),
    "spmvk_nccl_group_end": (cint, []),
    "spmvk_nccl_iter_create": (cint, [vp, vp, u64, u64, u64, u64, cint, C.POINTER(vp)]),
    "spmvk_nccl_iter_x": (cint, [vp, cint, C.POINTER(vp), u64p]),
    "spmvk_nccl_iter_current": (cint, [vp, C.POINTER(cint)]),
    "spmvk_nccl_iter_halo_entries": (cint, [vp, u64p]),
    "spmvk_nccl_iter_step_f64": (cint, [vp, C.c_double, vp, vp]),
    "spmvk_nccl_iter_step_f32": (cint, [vp, C.c_float, vp, vp]),
    "spmvk_nccl_iter_destroy": (None, [vp]),
    "spmvk_dist_set_timeout_ms": (cint, [vp, u64]),
    "spmvk_dist_status": (cint, [vp, vp]),
    "spmvk_dist_destroy": (None, [vp]),
    "spmvk_gen_random_vector": (None, [u64, u64, vp]),
    "spmvk_gen_stencil": (u64, [cint, u64, vp, vp, vp]),
    "spmvk_gen_powerlaw": (u64, [u64, u64, vp, vp, vp]),
    "spmvk_gen_random_rows": (u64, [u64, u64, u64, u64, vp, vp, vp]),
    "spmvk_gen_block": (u64, [u64, u64, u64, u64, vp, vp, vp]),
    "spmvk_gen_banded": (u64, [u64, u64, u64, vp, vp, vp]),
}

_lib = None
_lock = threading.Lock()


class LibraryMissing(RuntimeError):
    pass


def lib():
    """The loaded libspmvk.so with every signature bound (loads once)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissing(
                    f"{LIB_PATH} is not built; run __graft_entry__.build() "
                    "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def last_error() -> str:
    m = lib().spmvk_last_error()
    return m.decode() if m else ""
