"""ctypes binding of the C ABI in include/ozb200.h.

This is the only place the package touches the native library.  There is no
CPU fallback: if libozb200.so is missing or no CUDA device is present, every
compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import STATUS_TO_ERROR, DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
# OZ_LIB_PATH selects an alternative in-tree build (A/B tuning of kernel variants)
LIB_PATH = os.environ.get("OZ_LIB_PATH") or os.path.join(_HERE, "libozb200.so")

_i64 = C.c_int64
_i32 = C.c_int32
_int = C.c_int
_dbl = C.c_double
_vp = C.c_void_p
_u64 = C.c_uint64

# name -> argtypes (restype is always int status unless listed in _RESTYPES)
_SIGNATURES = {
    "oz_version": [],
    "oz_launch_count": [],
    "oz_prof_enable": [_int],
    "oz_prof_summary": [_vp],
    "oz_sm_count": [_vp],
    "oz_split_aux_bytes": [],
    "oz_split": [_vp, _i64, _i64, _i64, _i64, _int, _int, _int, _int, _vp, _i64, _i64, _vp, _vp,
                 _vp],
    "oz_gemm_emu": [_i64, _i64, _i64, _vp, _i64, _i64, _int, _vp, _vp, _i64, _i64, _int, _vp,
                    _int, _vp, _vp, _vp, _int, _dbl, _dbl, _vp, _i64, _int, _vp, _vp],
    "oz_axpby": [_i64, _dbl, _vp, _dbl, _vp, _int, _vp, _vp],
    "oz_plan_groups": [_int, _vp, _i64, _int, _vp, _vp],
    "oz_gemm_pair_i32": [_i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp],
    "oz_dgemm": [_int, _int, _i64, _i64, _i64, _dbl, _vp, _i64, _vp, _i64, _dbl, _vp, _i64, _vp],
    "oz_lu_workspace_bytes": [_i64, _i64, _int, _int],
    "oz_lu_factor": [_vp, _i64, _i64, _i64, _int, _int, _int, _int, _vp, _vp, _vp, _vp, _vp,
                     _vp, _vp, C.c_size_t, _vp],
    "oz_lu_factor_overlapped": [_vp, _i64, _i64, _i64, _int, _int, _int, _int, _vp, _vp, _vp,
                                _vp, _vp, _vp, _vp, C.c_size_t, _vp, _i64, _vp],
    "oz_memcpy2d_h2d": [_vp, C.c_size_t, _vp, C.c_size_t, C.c_size_t, C.c_size_t, _vp],
    "oz_nonfinite_flag": [_vp, _i64, _i64, _i64, _i64, _vp, _vp],
    "oz_ipiv_to_perm": [_vp, _i64, _vp],
    "oz_lu_solve": [_vp, _i64, _i64, _vp, _vp, _vp, _vp, C.c_size_t, _vp],
    "oz_lu_solve_workspace_bytes": [_i64],
    "oz_residual_norms": [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp],
    "oz_row_sums": [_vp, _i64, _i64, _i64, _vp, _vp],
    "oz_max_abs": [_vp, _i64, _i64, _i64, _i64, _vp, _vp],
    "oz_generate": [_int, _i64, _i64, _i64, _dbl, _u64, _u64, _u64, _u64, _vp, _i64, _i64, _vp],
    "oz_copy2d": [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _vp],
    # step-level LU (distributed driver, hpl.py)
    "oz_lu_ws_init": [_vp, C.c_size_t, _i64, _i64, _int, _vp],
    "oz_lu_panel": [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, C.c_size_t, _i64, _i64,
                    _int, _int, _vp],
    "oz_laswp": [_vp, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _int, _vp, C.c_size_t, _i64, _i64,
                 _int, _vp],
    "oz_trsm_lunit": [_vp, _i64, _i64, _vp, _i64, _i64, _vp],
    "oz_schur_update": [_int, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int, _int, _int,
                        _vp, _vp, _vp, _vp, _vp, C.c_size_t, _i64, _i64, _vp],
    "oz_max_abs_bits": [_vp, _i64, _i64, _i64, _i64, _int, _vp, _vp],
    "oz_schur_split": [_int, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _int, _int, _vp, C.c_size_t,
                       _i64, _i64, _vp],
    "oz_schur_cols": [_int, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int, _int, _int,
                      _vp, _vp, _vp, _vp, _i64, _i64, _int, _vp, C.c_size_t, _i64, _i64, _vp],
    "oz_trsv_block": [_vp, _i64, _i64, _int, _vp, _vp, _vp, C.c_size_t, _vp],
    "oz_gemv_partial": [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp],
    "oz_generate_cyclic": [_int, _i64, _i64, _i64, _dbl, _u64, _u64, _u64, _u64, _i64, _i64,
                           _i64, _i64, _vp, _i64, _vp],
    "oz_generate_block_cyclic": [_int, _i64, _i64, _i64, _dbl, _u64, _u64, _u64, _u64, _i64,
                                 _i64, _i64, _i64, _i64, _i64, _i64, _vp, _i64, _vp],
    "oz_dpanel_candidate": [_vp, _i64, _i64, _i64, _int, _int, _int, _i64, _i64, _i64, _vp, _vp],
    "oz_dpanel_apply": [_vp, _i64, _i64, _i64, _int, _int, _i64, _int, _i64, _i64, _i64, _vp,
                        _vp, _vp, _vp, _vp],
    "oz_gather_rows": [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _vp],
    "oz_scatter_rows": [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _vp],
    "oz_scatter_vec": [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp],
    "oz_assemble_rows": [_vp, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _i64, _vp],
    "oz_gemm_starts_dump": [],
    "oz_panel_debug_counters": [_vp],
    "oz_lookahead_sms": [_i64, _i64, _i64, _int],
    "oz_lookahead_cols1": [_i64, _i64, _i64, _int, _int],
}
_RESTYPES = {
    "oz_launch_count": C.c_longlong,
    "oz_lookahead_sms": C.c_int,
    "oz_lookahead_cols1": C.c_int64,
    "oz_split_aux_bytes": C.c_size_t,
    "oz_lu_workspace_bytes": C.c_size_t,
    "oz_lu_solve_workspace_bytes": C.c_size_t,
    "oz_last_error": C.c_char_p,
}

_lock = threading.Lock()
_lib = None


def load() -> C.CDLL:
    """Load libozb200.so (once) and declare every exported signature."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_2509_23565_b200/csrc)"
            )
        lib = C.CDLL(LIB_PATH)
        lib.oz_last_error.restype = C.c_char_p
        lib.oz_last_error.argtypes = []
        for name, args in _SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None:
                raise DeviceError(f"{LIB_PATH} is stale: missing symbol {name}; rebuild it")
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    return ["oz_last_error", *_SIGNATURES.keys()]


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point; map failures onto errors.py."""
    lib = load()
    status = getattr(lib, name)(*args)
    if status != 0:
        msg = (lib.oz_last_error() or b"").decode(errors="replace")
        raise STATUS_TO_ERROR.get(status, DeviceError)(f"{name}: {msg}")


def query(name: str, *args):
    """Invoke a value-returning entry point (sizes)."""
    return getattr(load(), name)(*args)


def require_cuda():
    """Return torch after checking a CUDA device is present (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: this package has no CPU fallback")
    load()
    return torch


def ptr(t) -> int:
    return t.data_ptr()


def stream_handle(torch_mod=None) -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream
