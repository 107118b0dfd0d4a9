"""ctypes binding of include/terralio_gpu.h (the C-ABI boundary).

This is the binding a Python caller of the reference would add (see
INTEGRATION.md). It loads the in-tree libterralio_gpu.so and fails loudly when
it is missing: there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(os.environ.get("TLG_LIB_OVERRIDE") or
                 Path(__file__).resolve().parent / "lib" / "libterralio_gpu.so")

TLG_OK = 0
TLG_INVALID_ARGUMENT = 1
TLG_DOMAIN_ERROR = 2
TLG_NO_SUPPORTED_CENTERS = 3
TLG_RUNTIME_ERROR = 4
TLG_CUDA_ERROR = 5
TLG_OUT_OF_MEMORY = 6
TLG_BUFFER_TOO_SMALL = 7

TLG_HOST = 0
TLG_DEVICE = 1


class TerralioError(RuntimeError):
    """Base of all errors raised through the C-ABI."""


class InvalidArgument(TerralioError, ValueError):
    """std::invalid_argument in the reference."""


class DomainError(TerralioError, ValueError):
    """std::domain_error in the reference."""


class NoSupportedCenters(TerralioError):
    """terrain::NoSupportedCenters (center_select.hpp:30-32)."""


class CudaError(TerralioError):
    pass


class OutOfMemory(TerralioError, MemoryError):
    pass


class BufferTooSmall(TerralioError, BufferError):
    pass


_STATUS_EXC = {
    TLG_INVALID_ARGUMENT: InvalidArgument,
    TLG_DOMAIN_ERROR: DomainError,
    TLG_NO_SUPPORTED_CENTERS: NoSupportedCenters,
    TLG_RUNTIME_ERROR: TerralioError,
    TLG_CUDA_ERROR: CudaError,
    TLG_OUT_OF_MEMORY: OutOfMemory,
    TLG_BUFFER_TOO_SMALL: BufferTooSmall,
}


class KernelParamsC(C.Structure):
    _fields_ = [("sigma", C.c_double), ("sigma_eps", C.c_double), ("lambda_", C.c_double),
                ("cutoff_radius", C.c_double)]


class CenterParamsC(C.Structure):
    _fields_ = [("mesh_resolution", C.c_double), ("accept_radius", C.c_double),
                ("accept_count", C.c_int32), ("reserved", C.c_int32),
                ("roi_min_x", C.c_double), ("roi_min_y", C.c_double),
                ("roi_max_x", C.c_double), ("roi_max_y", C.c_double)]


class UpdateReportC(C.Structure):
    _fields_ = [("active_blocks", C.c_uint64), ("active_centers", C.c_uint64),
                ("born_centers", C.c_uint64), ("rejected", C.c_int32), ("solver", C.c_int32),
                ("flops", C.c_double)]


class NormalEqC(C.Structure):
    _fields_ = [("A", C.c_double * 21), ("g", C.c_double * 6), ("cost", C.c_double),
                ("valid", C.c_double)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_SZ = C.c_size_t
_I = C.c_int
_ST = C.c_int

# name -> (restype, argtypes)
_SIGS = {
    "tlg_abi_version": (C.c_int, []),
    "tlg_last_error": (C.c_char_p, []),
    "tlg_ctx_create": (_ST, [_I, _P, C.POINTER(_P)]),
    "tlg_ctx_destroy": (_ST, [_P]),
    "tlg_ctx_set_stream": (_ST, [_P, _P]),
    "tlg_ctx_synchronize": (_ST, [_P]),
    "tlg_ctx_launch_count": (C.c_uint64, [_P]),
    "tlg_ctx_set_profiling": (_ST, [_P, _I]),
    "tlg_ctx_kernel_stats": (_ST, [_P, _I, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
    "tlg_lm_step": (_ST, [_P, _P, C.c_double, _P]),
    "tlg_ne_min_eigenvalue": (_ST, [_P, _P, C.POINTER(C.c_double)]),
    "tlg_match_config_default": (_ST, [_P]),
    "tlg_map_create": (_ST, [_P, C.c_double, _SZ, _P]),
    "tlg_map_destroy": (_ST, [_P]),
    "tlg_map_insert": (_ST, [_P, _P, _P, _P, _P, _P, _SZ, _I, _P, _P]),
    "tlg_map_points": (_ST, [_P, _I, _P, _P, _SZ, C.POINTER(_SZ)]),
    "tlg_build_correspondences": (_ST, [_P, _P, _P, _P, _P, _SZ, _I, _P, _P, _P, C.POINTER(_SZ)]),
    "tlg_correspondences_get": (_ST, [_P, _P, _P, _P, _P, _P, _P, _P, _SZ]),
    "tlg_feature_normal_eq": (_ST, [_P, _P, _P, _P]),
    "tlg_batch_ridge_pattern": (_ST, [_P, C.POINTER(_SZ)]),
    "tlg_batch_ridge_pack": (_ST, [_P, _P, _P]),
    "tlg_batch_ridge_unpack": (_ST, [_P, _P, _P]),
    "tlg_comm_unique_id": (_ST, [_P]),
    "tlg_comm_init": (_ST, [_P, _P, _I, _I, C.POINTER(_P)]),
    "tlg_comm_destroy": (_ST, [_P]),
    "tlg_comm_allreduce_normal_eq": (_ST, [_P, _P]),
    "tlg_fit_batch_ridge_sharded": (_ST, [_P, _P, _P, _P, _P, _SZ, _I]),
    "tlg_feature_rows": (_ST, [_P, _P, _P, _P, _P, _SZ, _P, _P, _P, _P, _SZ, C.POINTER(_SZ)]),
    "tlg_select_ground_points": (_ST, [_P, _P, _P, _P, _P, _SZ, _I, _P, _P, _P, _P, C.c_double,
                                       C.c_double, _SZ, _P, _P, _P, _I, C.POINTER(_SZ)]),
    "tlg_terrain_error_histogram": (_ST, [_P, _P, _P, _P, _SZ, _I, C.c_double, _I, _P, _P,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "tlg_kernel_finalize": (_ST, [C.POINTER(KernelParamsC)]),
    "tlg_kernel_eval": (_ST, [_P, C.POINTER(KernelParamsC), _P, _P, _P, _P, _SZ, _I, C.c_double,
                              _P, _I]),
    "tlg_supported_mesh_nodes": (_ST, [_P, _P, _P, _P, _SZ, _SZ, _I, C.POINTER(CenterParamsC),
                                       _P, _P, _SZ, C.POINTER(_SZ), _I]),
    "tlg_select_centers": (_ST, [_P, _P, _P, _P, _SZ, _SZ, _I, C.POINTER(CenterParamsC),
                                 _P, _P, _SZ, C.POINTER(_SZ), _I]),
    "tlg_model_create": (_ST, [_P, C.POINTER(KernelParamsC), C.POINTER(CenterParamsC), _P, _P,
                               _SZ, _I, C.POINTER(_P)]),
    "tlg_model_destroy": (_ST, [_P]),
    "tlg_model_counts": (_ST, [_P, C.POINTER(_SZ), C.POINTER(_SZ)]),
    "tlg_model_sweep": (_ST, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "tlg_model_set_exact_cutoff": (_ST, [_P, C.c_int]),
    "tlg_model_kernel": (_ST, [_P, C.POINTER(KernelParamsC)]),
    "tlg_model_center_params": (_ST, [_P, C.POINTER(CenterParamsC)]),
    "tlg_model_get_centers": (_ST, [_P, _P, _P, _I]),
    "tlg_model_get_weights": (_ST, [_P, _P, _I]),
    "tlg_model_set_weights": (_ST, [_P, _P, _I]),
    "tlg_model_get_block_index": (_ST, [_P, _P, _I]),
    "tlg_model_block_size": (_ST, [_P, C.c_uint32, C.POINTER(_SZ)]),
    "tlg_model_get_block_members": (_ST, [_P, C.c_uint32, _P]),
    "tlg_model_get_block_info_inverse": (_ST, [_P, C.c_uint32, _P, _I]),
    "tlg_model_set_block_info_inverse": (_ST, [_P, C.c_uint32, _P, _I]),
    "tlg_eval": (_ST, [_P, _P, _P, _SZ, _I, _P, _P, _P, _P, _I]),
    "tlg_moment_features": (_ST, [_P, _P, _P, _SZ, _I, _P, _P, _P, _SZ, C.POINTER(_SZ), _I]),
    "tlg_manifold_rows": (_ST, [_P, _P, _P, _P, _P, _P, _SZ, _I, C.c_double, C.c_double,
                                C.c_double, _P, _P, _P, _P, _I, C.POINTER(NormalEqC)]),
    "tlg_scan_create": (_ST, [_P, _P, _P, _P, _P, _P, _SZ, _I, C.POINTER(_P)]),
    "tlg_scan_destroy": (_ST, [_P]),
    "tlg_scan_info": (_ST, [_P, C.POINTER(_SZ), C.POINTER(C.c_double)]),
    "tlg_scan_permutation": (_ST, [_P, _P, _I]),
    "tlg_scan_manifold_rows": (_ST, [_P, _P, _P, _P, C.c_double, C.c_double, C.c_double, _P, _P,
                                     _P, _P, _I, C.POINTER(NormalEqC)]),
    "tlg_recursive_update": (_ST, [_P, _P, _P, _P, _SZ, _SZ, _I, _I, C.POINTER(UpdateReportC)]),
    "tlg_batch_ridge_system": (_ST, [_P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                     C.POINTER(C.c_size_t)]),
    "tlg_batch_ridge_assemble": (_ST, [_P, _P, _P, _P, C.c_size_t, C.c_int, _P, C.c_size_t, _P,
                                       C.c_int]),
    "tlg_batch_ridge_solve": (_ST, [_P, _P, C.c_size_t, _P]),
    "tlg_fit_batch_ridge": (_ST, [_P, C.POINTER(KernelParamsC), C.POINTER(CenterParamsC), _P, _P,
                                  _SZ, _P, _P, _P, _SZ, _SZ, _I, C.POINTER(_P)]),
    "tlg_model_save": (_ST, [_P, C.c_char_p]),
    "tlg_model_load": (_ST, [_P, C.c_char_p, C.POINTER(_P)]),
}

_lib = None


def lib_path() -> Path:
    return _LIB_PATH


def load() -> C.CDLL:
    """Loads libterralio_gpu.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -m paper_2509_26222_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.tlg_abi_version() != 1:
        raise ImportError("terralio_gpu ABI version mismatch")
    _lib = lib
    return lib


_diag = None


def load_diag() -> C.CDLL:
    """Loads libterralio_diag.so: DIAGNOSTICS, not the product ABI
    (include/terralio_diag.h: FP64 peak microbenchmark, dense-layer hooks)."""
    global _diag
    if _diag is None:
        load()
        path = _LIB_PATH.parent / "libterralio_diag.so"
        d = C.CDLL(str(path))
        d.tlg_diag_fp64_peak.restype = C.c_int
        d.tlg_diag_fp64_peak.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        d.tlg_diag_dense_bench.restype = C.c_int
        d.tlg_diag_dense_bench.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(C.c_double)]
        d.tlg_diag_potrf.restype = C.c_int
        d.tlg_diag_potrf.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                     C.c_void_p]
        d.tlg_diag_set_batch_gram.restype = C.c_int
        d.tlg_diag_set_batch_gram.argtypes = [C.c_void_p, C.c_int]
        d.tlg_diag_last_gram_lattice.restype = C.c_int
        d.tlg_diag_last_gram_lattice.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
        _diag = d
    return _diag


def exported_symbols() -> list[str]:
    return list(_SIGS)


def check(status: int) -> None:
    if status == TLG_OK:
        return
    msg = (load().tlg_last_error() or b"").decode(errors="replace")
    raise _STATUS_EXC.get(status, TerralioError)(msg)
