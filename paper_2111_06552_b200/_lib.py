"""ctypes binding of libgcgb200.so (the C ABI in include/gcgb200.h).

The library is the only compute path of this package: if it is missing, or
there is no CUDA device, every entry point raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import GcgError, InvalidShape, NoConvergence

_HERE = os.path.dirname(os.path.abspath(__file__))
# GCG_LIB_ALT (development A/B only): another build of the same library next to this file
LIB_PATH = os.path.join(_HERE, os.environ.get("GCG_LIB_ALT") or "libgcgb200.so")

_i64, _i32, _dbl, _ptr, _int = C.c_int64, C.c_int32, C.c_double, C.c_void_p, C.c_int

# name -> argtypes (all return int status unless listed in _RESTYPE)
_SIGS = {
    "gcg_abi_version": [],
    "gcg_status_string": [_int],
    "gcg_launch_count": [],
    "gcg_cusolver_calls": [],
    "gcg_nccl_available": [],
    "gcg_coo_to_csr": [_ptr, _i64, _i64, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, C.POINTER(_i64)],
    "gcg_nccl_unique_id": [_ptr],
    "gcg_nccl_comm_create": [_ptr, _i32, _i32, _ptr, C.POINTER(_ptr)],
    "gcg_nccl_comm_destroy": [_ptr],
    "gcg_nccl_allreduce_sum": [_ptr, _ptr, _ptr, _i64],
    "gcg_ctx_create": [C.POINTER(_ptr), _ptr],
    "gcg_ctx_destroy": [_ptr],
    "gcg_ctx_set_stream": [_ptr, _ptr],
    "gcg_ctx_sync": [_ptr],
    "gcgeig_csr_matvec": [_ptr, _ptr, _ptr, _i64, _i64, _ptr, _i64, _i64, _ptr, _i64],
    "gcgeig_csr_create": [_ptr, _ptr, _ptr, _i64, _i64, C.POINTER(_ptr)],
    "gcgeig_csr_apply": [_ptr, _ptr, _i64, _i64, _ptr, _i64],
    "gcgeig_csr_destroy": [_ptr],
    "gcgeig_inner_product": [_ptr, _i64, _i64, _i64, _ptr, _i64, _i64, _ptr, _i64, _i64, _i64, _int],
    "gcgeig_axpby": [_dbl, _ptr, _i64, _i64, _i64, _dbl, _ptr, _i64],
    "gcg_prof_begin": [_ptr],
    "gcg_prof_end": [_ptr, _ptr],
    "gcg_prof_sample": [_ptr, _int],
    "gcg_spmm_csr": [_ptr, _i64, _i64, _ptr, _ptr, _ptr, _i64, _ptr, _i64, _dbl, _dbl, _ptr, _i64,
                     _dbl, _ptr, _i64, _ptr, _i64, _int, _ptr, _i64, _ptr],
    "gcg_build_p": [_ptr, _i64, _i64, _ptr, _i64, _i64, _i64, _i64, _dbl, _ptr, _i64,
                    C.POINTER(_i64)],
    "gcg_sell_size": [_ptr, _i64, _ptr, _i32, C.POINTER(_i64), C.POINTER(_i64)],
    "gcg_csr_to_sell": [_ptr, _i64, _ptr, _ptr, _ptr, _i32, _ptr, _ptr, _ptr, _ptr],
    "gcg_spmm_sell": [_ptr, _i64, _i64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _i64, _dbl, _dbl, _ptr,
                      _i64, _dbl, _ptr, _i64, _ptr, _i64, _int, _ptr, _i64, _ptr],
    "gcg_gram": [_ptr, _i64, _i64, _i64, _ptr, _i64, _ptr, _i64, _dbl, _dbl, _ptr, _i64, _i64, _ptr,
                 _i64, _ptr],
    "gcg_lincomb": [_ptr, _i64, _i64, _i64, _dbl, _ptr, _i64, _ptr, _i64, _dbl, _ptr, _i64],
    "gcg_axpby": [_ptr, _i64, _i64, _dbl, _ptr, _i64, _dbl, _ptr, _i64],
    "gcg_copy": [_ptr, _i64, _i64, _ptr, _i64, _ptr, _i64],
    "gcg_col_scale": [_ptr, _i64, _i64, _ptr, _ptr, _i64],
    "gcg_col_dots": [_ptr, _i64, _i64, _ptr, _i64, _ptr, _i64, _ptr],
    "gcg_fill": [_ptr, _i64, _i64, _dbl, _ptr, _i64],
    "gcg_block_cg": [_ptr, _i64, _i64, _ptr, _ptr, _ptr, _dbl, _i64, _ptr, _i64, _ptr, _i64, _i32,
                     _dbl, _ptr, _ptr, _ptr, _ptr],
    "gcg_block_cg_x0": [_ptr, _i64, _i64, _ptr, _ptr, _ptr, _dbl, _i64, _ptr, _i64, _ptr, _i64,
                        _ptr, _i64, _i32, _dbl, _ptr, _ptr, _ptr, _ptr],
    "gcg_col_scale_copy": [_ptr, _i64, _i64, _ptr, _ptr, _i64, _ptr, _i64],
    "gcg_block_cg_dist": [_ptr, _i64, _i64, _ptr, _ptr, _ptr, _dbl, _i64, _ptr, _i64, _ptr, _i64,
                          _i32, _dbl, _ptr, _ptr, _ptr, _ptr, _ptr],
    "gcg_gather_rows": [_ptr, _i64, _ptr, _i64, _ptr, _i64, _ptr, _i64],
    "gcg_fp64_peak": [_ptr, _int, _i32, C.POINTER(C.c_double), _ptr],
    "gcg_ritz_sums": [_ptr, _i64, _i64, _ptr, _i64, _ptr, _i64, _ptr, _i64, _ptr, _int, _ptr],
    "gcg_ritz_finish": [_ptr, _i64, _ptr, _ptr, _int, _ptr],
    "gcg_syev": [_ptr, _i64, _ptr, _i64, _ptr, _ptr, _i64],
    "gcg_syev_range": [_ptr, _i64, _ptr, _i64, _i64, _i64, _ptr, _ptr, _i64],
    "gcg_dgemm": [_ptr, _int, _int, _i64, _i64, _i64, _dbl, _ptr, _i64, _ptr, _i64, _dbl, _ptr,
                  _i64],
    "gcg_symmetrize": [_ptr, _i64, _ptr, _i64],
    "gcg_svqb_prepare": [_ptr, _i64, _ptr, _i64, _dbl, _dbl, _ptr, _i64, _ptr],
    "gcg_deflate_status": [_ptr, _i64, _i64, _ptr, _i64, _ptr, _i64, _dbl, _ptr],
    "gcg_abar_assemble": [_ptr, _i64, _i64, _i64, _ptr, _ptr, _i64, _ptr, _i64, _ptr, _i64],
    "gcg_max_abs_diff": [_ptr, _i64, _i64, _ptr, _i64, _ptr, _i64, _ptr],
    "gcg_count_le": [_ptr, _i64, _ptr, _dbl, _ptr],
    "gcg_scale_rsqrt": [_ptr, _i64, _i64, _ptr, _i64, _ptr, _ptr, _i64],
    "gcg_ritz_residuals": [_ptr, _i64, _i64, _ptr, _i64, _ptr, _i64, _ptr, _i64, _ptr, _int, _ptr],
    "gcg_orth_recursive": [_ptr, _i64, _ptr, _i64, _i64, _i64, _i64, _ptr, _ptr, _ptr, _ptr,
                           _ptr, _ptr, _ptr, _i64, _ptr],
    "gcg_orth_against": [_ptr, _i64, _ptr, _i64, _i64, _ptr, _i64, _i64, _i64, _ptr, _ptr, _ptr,
                         _ptr, _ptr, _ptr, _ptr, _i64, _ptr],
    "gcg_stencil_nnz": [_i64, _i64, _i64, _i32, _ptr, _ptr],
    "gcg_stencil_csr": [_ptr, _i64, _i64, _i64, _i32, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr],
    "gcg_varcoef7_weights": [_ptr, _i64, _ptr, _ptr],
    "gcg_stencil_slab": [_ptr, _i64, _i64, _i64, _i32, _ptr, _ptr, _ptr, _i64, _i64, _ptr, _ptr,
                         _ptr, C.POINTER(_i64)],
    "gcg_csr_check": [_ptr, _i64, _ptr, _ptr, _ptr, _ptr],
    "gcg_fill_normal": [_ptr, _i64, _i64, _i64, C.c_uint64, _ptr, _i64],
    "gcg_mm_open": [C.c_char_p, _int, C.POINTER(_ptr), _ptr],
    "gcg_mm_fetch": [_ptr, _ptr, _ptr, _ptr],
    "gcg_mm_close": [_ptr],
}
_RESTYPE = {"gcg_status_string": C.c_char_p, "gcg_launch_count": _i64, "gcg_cusolver_calls": _i64, "gcg_mm_close": None}


class OrthOpts(C.Structure):
    """gcg_orth_opts (include/gcgb200.h)."""

    _fields_ = [
        ("svd_leaf", C.c_int64),
        ("reorth_tol", C.c_double),
        ("dependence_tol", C.c_double),
        ("max_passes", C.c_int32),
        ("pad_", C.c_int32),
    ]


class MMInfo(C.Structure):
    """gcg_mm_info (include/gcgb200.h)."""

    _fields_ = [
        ("nrows", C.c_int64),
        ("ncols", C.c_int64),
        ("nentries", C.c_int64),
        ("format", C.c_int32),
        ("symmetric", C.c_int32),
        ("err_kind", C.c_int32),
        ("pad_", C.c_int32),
        ("err_line", C.c_int64),
        ("err_msg", C.c_char * 240),
    ]

EXPORTED = tuple(_SIGS)

# int (*callback)(int op, int k, void* user) of gcg_cg_dist
CG_DIST_CALLBACK = C.CFUNCTYPE(C.c_int, C.c_int, C.c_int, C.c_void_p)


class CgDist(C.Structure):
    """gcg_cg_dist (include/gcgb200.h)."""

    _fields_ = [
        ("nghost", C.c_int64),
        ("nsend", C.c_int64),
        ("send_idx", C.c_void_p),
        ("send_buf", C.c_void_p),
        ("recv_buf", C.c_void_p),
        ("red_buf", C.c_void_p),
        ("callback", CG_DIST_CALLBACK),
        ("user", C.c_void_p),
        ("nccl_comm", C.c_void_p),
        ("npeer", C.c_int32),
        ("peer_rank", C.c_void_p),
        ("peer_send_off", C.c_void_p),
        ("peer_recv_off", C.c_void_p),
    ]

_lib = None


class LibraryMissing(GcgError):
    """libgcgb200.so is not built or cannot be loaded (no CPU fallback exists)."""


def load(path=LIB_PATH):
    """Load and type the shared library (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryMissing(
            f"{path} not found: build it with `python -m paper_2111_06552_b200.build`"
        )
    lib = C.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, _int)
    _lib = lib
    return lib


class DeviceError(GcgError):
    """A CUDA runtime error inside the library."""


def check(status, what=""):
    if status == 0:
        return
    msg = load().gcg_status_string(status).decode()
    text = f"{what}: {msg}" if what else msg
    if status == 1:
        raise InvalidShape(text)
    if status == 3:
        raise NoConvergence(text)
    raise DeviceError(text)


def call(name, *args):
    check(getattr(load(), name)(*args), name)


def launch_count():
    return int(load().gcg_launch_count())


def cusolver_calls():
    """cuSOLVER eigensolver calls since load (none for Rayleigh-Ritz orders <= 1024)."""
    return int(load().gcg_cusolver_calls())
