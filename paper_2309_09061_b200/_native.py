"""ctypes binding of libh2g.so (include/h2g.h).

The library is built in-tree (paper_2309_09061_b200/libh2g.so) by __graft_entry__.build() /
`make -C paper_2309_09061_b200/csrc`.  There is no CPU fallback: every product entry point
raises if the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import CudaError, InvalidInputError, StructureError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libh2g.so")
# H2G_LIB: an alternative build of the same library (A/B timing of engine changes, tools/ab.sh)
LIB_PATH = os.environ.get("H2G_LIB", LIB_PATH)

_lib = None

P = C.c_void_p
I64P = C.POINTER(C.c_longlong)
F64P = C.POINTER(C.c_double)
U8P = C.POINTER(C.c_ubyte)

SIGNATURES = {
    "h2g_ctx_create": (C.c_int, [C.c_int, P, C.POINTER(P)]),
    "h2g_matvec": (C.c_int, [P, P, C.c_int, P, P, C.c_double, C.c_int]),
    "h2g_h2_build_kernel": (C.c_int, [P, P, C.c_int, C.c_int, F64P, F64P, I64P, I64P, I64P, F64P, C.c_longlong,
                                      I64P, F64P, C.c_longlong, C.POINTER(P)]),
    "h2g_ctx_destroy": (C.c_int, [P]),
    "h2g_ctx_set_timing": (C.c_int, [P, C.c_int]),
    "h2g_ctx_stage_times": (C.c_int, [P, F64P]),
    "h2g_ctx_stage_times_ext": (C.c_int, [P, F64P, C.c_int]),
    "h2g_ctx_mem": (C.c_int, [P, I64P, C.c_int]),
    "h2g_ctx_set_alltoall": (C.c_int, [P, P, P]),
    "h2g_ctx_counters": (C.c_int, [P, I64P, C.c_int]),
    "h2g_ctx_synchronize": (C.c_int, [P]),
    "h2g_ctx_host_times": (C.c_int, [P, C.c_char_p, C.c_int, C.c_int]),
    "h2g_ctx_set_profile": (C.c_int, [P, C.c_int]),
    "h2g_set_serial": (C.c_int, [C.c_int]),
    "h2g_ctx_kernel_stats": (C.c_int, [P, F64P, C.c_int]),
    "h2g_ctx_trace_begin": (C.c_int, [P]),
    "h2g_ctx_trace_dump": (C.c_int, [P, C.c_char_p]),
    "h2g_ctx_set_comm": (C.c_int, [P, C.c_int, C.c_int, C.c_void_p, P]),
    "h2g_tree_partition": (C.c_int, [P, C.c_int, I64P, C.POINTER(C.c_int)]),
    "h2g_tree_create": (C.c_int, [P, C.c_int, I64P, I64P, I64P, I64P, C.POINTER(P)]),
    "h2g_tree_destroy": (None, [P]),
    "h2g_blocks_create": (C.c_int, [P, P, P, C.c_int, I64P, I64P, I64P, I64P, U8P, C.POINTER(P)]),
    "h2g_blocks_destroy": (None, [P]),
    "h2g_h2_upload": (C.c_int, [P, P, I64P, I64P, I64P, F64P, C.c_longlong, I64P, I64P, I64P, F64P,
                                C.c_longlong, C.c_int, I64P, F64P, C.c_longlong, I64P, F64P, C.c_longlong,
                                C.POINTER(P)]),
    "h2g_h2_upload_async": (C.c_int, [P, P, I64P, I64P, I64P, F64P, C.c_longlong, I64P, I64P, I64P, F64P,
                                C.c_longlong, C.c_int, I64P, F64P, C.c_longlong, I64P, F64P, C.c_longlong,
                                C.POINTER(P)]),
    "h2g_h2_destroy": (None, [P]),
    "h2g_h2_sizes": (C.c_int, [P, I64P]),
    "h2g_h2_ranks": (C.c_int, [P, I64P, I64P]),
    "h2g_h2_structure": (C.c_int, [P, I64P, I64P, I64P, I64P, U8P]),
    "h2g_h2_download": (C.c_int, [P, P, I64P, I64P, I64P, F64P, I64P, I64P, I64P, F64P, I64P, F64P, I64P, F64P]),
    "h2g_product_tree": (C.c_int, [P, P, C.POINTER(P), I64P]),
    "h2g_blocks_structure": (C.c_int, [P, I64P, I64P, I64P, I64P, I64P, U8P]),
    "h2g_multiply": (C.c_int, [P, P, P, C.c_double, C.c_int, C.c_int, C.POINTER(P)]),
    "h2g_coarsen": (C.c_int, [P, P, P, C.c_double, C.c_int, C.c_int, C.POINTER(P)]),
    "h2g_coarsen_prefetch": (C.c_int, [P, P, P, C.c_double, C.c_int, C.c_int, F64P, C.c_longlong, C.POINTER(P)]),
    "h2g_recompress": (C.c_int, [P, P, C.c_double, C.c_int, C.POINTER(P)]),
    # stage-level entry points (include/h2g.h)
    "h2g_h2_basis": (C.c_int, [P, C.c_int, C.POINTER(P)]),
    "h2g_basis_upload": (C.c_int, [P, P, I64P, I64P, I64P, F64P, C.c_longlong, C.POINTER(P)]),
    "h2g_basis_sizes": (C.c_int, [P, I64P]),
    "h2g_basis_download": (C.c_int, [P, P, I64P, I64P, I64P, F64P]),
    "h2g_basis_destroy": (None, [P]),
    "h2g_mats_upload": (C.c_int, [P, C.c_int, I64P, I64P, I64P, F64P, C.c_longlong, C.POINTER(P)]),
    "h2g_mats_shapes": (C.c_int, [P, C.POINTER(C.c_int), I64P, I64P]),
    "h2g_mats_download": (C.c_int, [P, P, I64P, F64P]),
    "h2g_mats_destroy": (None, [P]),
    "h2g_cluster_basis_product": (C.c_int, [P, P, P, C.POINTER(P)]),
    "h2g_basis_weights": (C.c_int, [P, P, C.POINTER(P)]),
    "h2g_total_weights": (C.c_int, [P, P, C.c_int, P, C.c_int, C.POINTER(P)]),
    "h2g_compress_induced_row_basis": (C.c_int, [P, P, P, P, P, C.c_double, C.c_int, C.c_int, C.c_double,
                                                 C.POINTER(P)]),
    "h2g_compress_induced_col_basis": (C.c_int, [P, P, P, P, P, C.c_double, C.c_int, C.c_int, C.c_double,
                                                 C.POINTER(P)]),
    "h2g_induced_parts": (C.c_int, [P, C.POINTER(P), C.POINTER(P), C.POINTER(P)]),
    "h2g_induced_create": (C.c_int, [P, P, P, P, C.c_int, C.POINTER(P)]),
    "h2g_induced_destroy": (None, [P]),
    "h2g_assemble_product": (C.c_int, [P, P, P, P, P, P, C.POINTER(P)]),
    "h2g_block_norms": (C.c_int, [P, P, P, P]),
    "h2g_build_coarse_row_basis": (C.c_int, [P, P, P, C.c_double, C.c_int, C.c_int, P, P, C.POINTER(P)]),
    "h2g_build_coarse_col_basis": (C.c_int, [P, P, P, C.c_double, C.c_int, C.c_int, P, P, C.POINTER(P)]),
    "h2g_cstate_parts": (C.c_int, [P, C.POINTER(P), C.POINTER(P), C.POINTER(P), I64P]),
    "h2g_cstate_destroy": (None, [P]),
    "h2g_project_final": (C.c_int, [P, P, P, P, P, C.POINTER(P)]),
    "h2g_last_error": (C.c_char_p, []),
}


def load(path: str = LIB_PATH):
    """Load the native library and declare every exported symbol of include/h2g.h."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise CudaError(f"native library {path} is missing; run __graft_entry__.build()")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status == 0:
        return
    msg = load().h2g_last_error().decode()
    if status == 1:
        raise InvalidInputError(msg)
    if status == 2:
        raise StructureError(msg)
    raise CudaError(msg)


def i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(I64P)


def f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(F64P)


def u8(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return a, a.ctypes.data_as(U8P)
