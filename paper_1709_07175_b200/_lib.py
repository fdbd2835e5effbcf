"""ctypes binding of the C ABI declared in include/lazypca_b200.h.

Loads the in-tree liblazypca_b200.so. There is no fallback: if the library is
missing, or a compute call runs without an sm_100 device, the call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["LPCA_LIB_PATH"]) if os.environ.get("LPCA_LIB_PATH") else _PKG / "liblazypca_b200.so"
# (LPCA_LIB_PATH: another build of the same library, for A/B timing experiments)

LPCA_F32, LPCA_F64 = 4, 8
LPCA_HOST, LPCA_DEVICE = 0, 1
LPCA_ROW_MAJOR, LPCA_COL_MAJOR, LPCA_CSC = 0, 1, 2


class MatrixView(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("layout", C.c_int32), ("location", C.c_int32), ("reserved", C.c_int32),
        ("rows", C.c_int64), ("cols", C.c_int64), ("ld", C.c_int64),
        ("data", C.c_void_p), ("col_ptr", C.c_void_p), ("row_idx", C.c_void_p), ("nnz", C.c_int64),
    ]


class Config(C.Structure):
    _fields_ = [
        ("method", C.c_int32), ("projection_kind", C.c_int32),
        ("k", C.c_int64), ("l", C.c_int64), ("proj_n", C.c_int64), ("proj_l", C.c_int64),
        ("density", C.c_double), ("seed", C.c_uint64), ("block_rows", C.c_int64),
        ("streaming", C.c_int32), ("deterministic", C.c_int32), ("power_iters", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Timings(C.Structure):
    _fields_ = [(f, C.c_double) for f in
                ("sketch", "qr", "f_form", "svd", "total", "power", "transform", "h2d", "d2h",
                 "sketch_pass", "f_pass", "transform_pass", "power_pass")]


# int32_t (*lpca_allreduce_fn)(void* user, double* data, int64_t count, void* cuda_stream)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)

# int32_t (*lpca_next_block_fn)(void* user, lpca_matrix_view* block, int64_t* slice_index)
NEXT_BLOCK_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(MatrixView), C.POINTER(C.c_int64))


class ReconReport(C.Structure):
    _fields_ = [("spectral_error", C.c_double), ("frobenius_error", C.c_double),
                ("has_sigma_k_plus_1", C.c_int32), ("has_bound", C.c_int32),
                ("sigma_k_plus_1", C.c_double), ("bound", C.c_double)]


class MapInfo(C.Structure):
    _fields_ = [
        ("method", C.c_int32), ("reserved", C.c_int32),
        ("k", C.c_int64), ("l", C.c_int64), ("n", C.c_int64),
        ("seed", C.c_uint64), ("density", C.c_double), ("scale", C.c_double),
        ("has_singular_values", C.c_int32), ("reserved2", C.c_int32),
    ]


P = C.c_void_p
PP = C.POINTER(C.c_void_p)
I32, I64, U64, D = C.c_int32, C.c_int64, C.c_uint64, C.c_double
DP = C.POINTER(C.c_double)

# name -> (restype, argtypes); the list is also the symbol contract the CPU
# tests check against include/lazypca_b200.h.
SIGNATURES = {
    "lpca_last_error": (C.c_char_p, []),
    "lpca_last_error_index": (I64, []),
    "lpca_last_error_gap": (D, []),
    "lpca_abi_version": (I32, []),
    "lpca_ctx_create": (I32, [I32, PP]),
    "lpca_nccl_unique_id": (I32, [P]),
    "lpca_ctx_create_dist": (I32, [I32, I32, I32, P, PP]),
    "lpca_ctx_create_hooked": (I32, [I32, I32, I32, P, P, PP]),
    "lpca_debug_check_guards": (I64, [P, P, I64]),
    "lpca_debug_row_schedule": (I32, [P, P, I32, I64, I64, P, I64, P, P]),
    "lpca_ctx_destroy": (I32, [P]),
    "lpca_ctx_set_stream": (I32, [P, P]),
    "lpca_ctx_synchronize": (I32, [P]),
    "lpca_ctx_set_gemm_path": (I32, [P, I32]),
    "lpca_ctx_set_exact_order": (I32, [P, I32]),
    "lpca_ctx_launch_count": (I64, [P]),
    "lpca_config_resolve": (I32, [C.POINTER(Config), I64, C.POINTER(Config)]),
    "lpca_density_for": (I32, [I32, I64, D, DP]),
    "lpca_regenerate": (I32, [P, I32, I64, I64, D, U64, P, I32, DP]),
    "lpca_fit": (I32, [P, C.POINTER(Config), C.POINTER(MatrixView), PP, C.POINTER(Timings)]),
    "lpca_transform": (I32, [P, P, C.POINTER(MatrixView), P, I32, I32, I32, I64, C.POINTER(Timings)]),
    "lpca_fit_transform": (I32, [P, C.POINTER(Config), C.POINTER(MatrixView), PP, P, I32, I32, I32,
                                 I64, C.POINTER(Timings)]),
    "lpca_fit_stream": (I32, [P, C.POINTER(Config), P, P, PP, C.POINTER(Timings)]),
    "lpca_map_info_get": (I32, [P, C.POINTER(MapInfo)]),
    "lpca_map_copy_v": (I32, [P, P, I32]),
    "lpca_map_copy_sigma": (I32, [P, P]),
    "lpca_map_create": (I32, [P, C.POINTER(MapInfo), P, P, PP]),
    "lpca_map_destroy": (I32, [P]),
    "lpca_chordal_distance": (I32, [P, P, I64, I64, P, I64, I64, I32, DP]),
    "lpca_read_sparse_matrix_market": (I32, [C.c_char_p, PP]),
    "lpca_read_dense_matrix_market": (I32, [C.c_char_p, PP]),
    "lpca_read_dense_csv": (I32, [C.c_char_p, PP]),
    "lpca_matrix_file_info": (I32, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "lpca_matrix_file_copy": (I32, [P, P, P, P]),
    "lpca_matrix_file_view": (I32, [P, C.POINTER(MatrixView)]),
    "lpca_matrix_file_free": (None, [P]),
    "lpca_write_sparse_matrix_market": (I32, [C.c_char_p, I64, I64, P, P, P]),
    "lpca_write_dense_matrix_market": (I32, [C.c_char_p, I64, I64, P]),
    "lpca_write_dense_csv": (I32, [C.c_char_p, I64, I64, P]),
    "lpca_open_matrix_market_stream": (I32, [C.c_char_p, I64, PP]),
    "lpca_open_csv_stream": (I32, [C.c_char_p, I64, PP]),
    "lpca_file_stream_next": (I32, [P, C.POINTER(MatrixView), C.POINTER(C.c_int64)]),
    "lpca_file_stream_close": (None, [P]),
    "lpca_reconstruction_error": (I32, [P, C.POINTER(MatrixView), P, I64, I64, I32, I32, I64, I64, I32, I64,
                                        C.POINTER(ReconReport)]),
    "lpca_row_space_reconstruction_error": (I32, [P, C.POINTER(MatrixView), P, I64, I64, I32,
                                                  C.POINTER(ReconReport)]),
    "lpca_spectral_norm": (I32, [P, C.POINTER(MatrixView), DP]),
    "lpca_bound_value": (I32, [I64, I64, I64, I64, D, DP]),
    "lpca_distance_preservation": (I32, [P, C.POINTER(MatrixView), P, P, I64, C.c_uint64, C.POINTER(C.c_int64), P, P,
                                         P, P, P, DP, DP]),
    "lpca_map_save": (I32, [P, C.c_char_p]),
    "lpca_map_load": (I32, [P, C.c_char_p, PP]),
    "lpca_map_file_write": (I32, [C.c_char_p, C.POINTER(MapInfo), P, P]),
    "lpca_map_file_read": (I32, [C.c_char_p, C.POINTER(MapInfo), P, I64, P]),
    "lpca_spmm": (I32, [P, C.POINTER(MatrixView), P, I64, I32, P, I32]),
    "lpca_gemm_t": (I32, [P, P, I64, I64, I32, C.POINTER(MatrixView), P, I32]),
    "lpca_dense_aat": (I32, [P, P, I64, I64, I32, P]),
    "lpca_eigh": (I32, [P, P, I64, I32, P, P]),
    "lpca_eigh_jacobi": (I32, [P, P, I64, I32, P, P]),
    "lpca_ctx_set_eigensolver": (I32, [P, I32]),
    "lpca_truncated_svd_via_gram": (I32, [P, P, I64, I64, I64, I32, P, P, P]),
    "lpca_synth_lowrank": (I32, [P, I64, I64, I64, I64, D, D, U64, I32, P, I64]),
    "lpca_sketch_f32": (I32, [P, C.POINTER(MatrixView), P, I64, P, I64]),
    "lpca_gemm_t_f32": (I32, [P, P, I64, I64, C.POINTER(MatrixView), P]),
}

_lib = None


def load() -> C.CDLL:
    """Loads (once) the product library. Raises if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() or "
                "`python -m paper_1709_07175_b200.build` (there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
