"""ctypes binding of libpff_b200.so (include/pff_b200.h).

There is no fallback: if the library is missing, or no CUDA device is
present when a device entry point is called, this raises.
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# PFF_LIB: an alternative build of the same ABI (A/B experiments, tools/)
LIB_PATH = os.environ.get("PFF_LIB") or os.path.join(_HERE, "libpff_b200.so")

_c_dp = ctypes.c_void_p   # device pointers are passed as raw addresses
_i, _d, _i64 = ctypes.c_int, ctypes.c_double, ctypes.c_int64

# name -> (restype, argtypes); the exact exported surface of include/pff_b200.h
SIGNATURES = {
    "pff_abi_version": (_i, []),
    "pff_last_error": (ctypes.c_char_p, []),
    "pff_launch_counter": (_i64, []),
    "pff_set_option": (_i, [_i, _i]),
    "pff_level_create": (_i, [ctypes.POINTER(ctypes.c_void_p), _i, _i, _i, ctypes.c_void_p,
                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "pff_level_destroy": (_i, [ctypes.c_void_p]),
    "pff_level_n_scalar": (_i64, [ctypes.c_void_p]),
    "pff_level_n_cells": (_i64, [ctypes.c_void_p]),
    "pff_level_qcache_len": (_i64, [ctypes.c_void_p]),
    "pff_level_uses_sweep": (_i, [ctypes.c_void_p]),
    "pff_level_set_window": (_i, [ctypes.c_void_p, _i, _i]),
    "pff_level_window": (_i, [ctypes.c_void_p, ctypes.c_void_p]),
    "pff_level_bind": (_i, [ctypes.c_void_p, _c_dp, _c_dp, _c_dp, _c_dp]),
    "pff_level_refresh": (_i, [ctypes.c_void_p, ctypes.c_void_p]),
    "pff_apply": (_i, [ctypes.c_void_p, _i, _c_dp, _c_dp, _c_dp, ctypes.c_void_p]),
    "pff_apply_cheb": (_i, [ctypes.c_void_p, _i, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _d,
                            _d, ctypes.c_void_p]),
    "pff_apply_cheb_first": (_i, [ctypes.c_void_p, _i, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp,
                                  _d, _d, ctypes.c_void_p]),
    "pff_apply_cheb_ex": (_i, [ctypes.c_void_p, _i, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp,
                               _d, _d, _i, ctypes.c_void_p]),
    "pff_apply_emit": (_i, [ctypes.c_void_p, _i, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _d,
                            ctypes.c_void_p]),
    "pff_smooth_init": (_i, [ctypes.c_void_p, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _d,
                             ctypes.c_void_p]),
    "pff_smooth_init_ex": (_i, [ctypes.c_void_p, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _d, _i,
                                ctypes.c_void_p]),
    "pff_dense_matvec": (_i, [_i64, _i64, _c_dp, _c_dp, _c_dp, ctypes.c_void_p]),
    "pff_coarse_dense": (_i, [_i64, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, _c_dp, ctypes.c_void_p]),
    "pff_apply_rows": (_i, [ctypes.c_void_p, _i, _c_dp, _c_dp, _c_dp, _i, _i, ctypes.c_void_p]),
    "pff_apply_host": (_i, [ctypes.c_void_p, _i, _c_dp, _c_dp, _c_dp, _c_dp, _i, ctypes.c_void_p]),
    "pff_diagonal": (_i, [ctypes.c_void_p, _c_dp, _c_dp, _i, ctypes.c_void_p]),
    "pff_residual": (_i, [ctypes.c_void_p, _c_dp, _i, _i, ctypes.c_void_p]),
    "pff_cell_matrices": (_i, [ctypes.c_void_p, _c_dp, ctypes.c_void_p]),
    "pff_dense_jacobian": (_i, [ctypes.c_void_p, _c_dp, _c_dp, ctypes.c_void_p]),
    "pff_dgemm": (_i, [_i, _i, _i, _d, _c_dp, _i, _c_dp, _i, _d, _c_dp, _i, ctypes.c_void_p]),
    "pff_dmat_axpby": (_i, [_i, _i, _d, _c_dp, _i, _d, _c_dp, _c_dp, _i, ctypes.c_void_p]),
    "pff_dmat_diag": (_i, [_i, _c_dp, _c_dp, _i, ctypes.c_void_p]),
    "pff_recip": (_i, [_i64, _c_dp, _c_dp, _i, ctypes.c_void_p]),
    "pff_flags": (_i, [_i64, _c_dp, _c_dp, _c_dp, _i, ctypes.c_void_p]),
    "pff_lumped_mass": (_i, [ctypes.c_void_p, _c_dp, ctypes.c_void_p]),
    "pff_active_set": (_i, [_i64, _c_dp, _c_dp, _c_dp, _c_dp, _d, _c_dp, _c_dp, _c_dp,
                            ctypes.c_void_p]),
    "pff_prolongate": (_i, [ctypes.c_void_p, ctypes.c_void_p, _c_dp, _c_dp, _i, ctypes.c_void_p]),
    "pff_restrict": (_i, [ctypes.c_void_p, ctypes.c_void_p, _c_dp, _c_dp, _i, ctypes.c_void_p]),
    "pff_inject_f64": (_i, [ctypes.c_void_p, ctypes.c_void_p, _c_dp, _c_dp, _i, ctypes.c_void_p]),
    "pff_inject_u8": (_i, [ctypes.c_void_p, ctypes.c_void_p, _c_dp, _c_dp, ctypes.c_void_p]),
    "pff_cons": (_i, [ctypes.c_void_p, _i, _i, _c_dp, _c_dp, ctypes.c_void_p]),
    "pff_cheb_init": (_i, [_i64, _c_dp, _c_dp, _d, _c_dp, _c_dp, _i, ctypes.c_void_p]),
    "pff_cheb_step": (_i, [_i64, _c_dp, _c_dp, _d, _d, _c_dp, _c_dp, ctypes.c_void_p]),
    "pff_axpby": (_i, [_i64, _d, _c_dp, _d, _c_dp, ctypes.c_void_p]),
    "pff_div": (_i, [_i64, _c_dp, _c_dp, _d, _c_dp, ctypes.c_void_p]),
    "pff_mul": (_i, [_i64, _c_dp, _c_dp, _c_dp, ctypes.c_void_p]),
    "pff_reduce_scratch_len": (_i64, []),
    "pff_copy_components": (_i, [_c_dp, _c_dp, _i64, _i, _i64, ctypes.c_void_p]),
    "pff_lanczos_ranges": (_i, [_i, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p, _i, ctypes.c_void_p, _c_dp, _c_dp,
                                ctypes.c_void_p]),
    "pff_dot": (_i, [_i64, _c_dp, _c_dp, _c_dp, _c_dp, ctypes.c_void_p]),
    "pff_mgs": (_i, [_i64, _i, _c_dp, _i64, _c_dp, _c_dp, _c_dp, ctypes.c_void_p]),
    "pff_mgs_lowsync": (_i, [_i64, _i, _c_dp, _i64, _c_dp, _c_dp, _i64, _c_dp, _c_dp,
                             ctypes.c_void_p]),
    "pff_mdot": (_i, [_i64, _i, _c_dp, _i64, _c_dp, _c_dp, _c_dp, ctypes.c_void_p]),
    "pff_combine": (_i, [_i64, _i, _c_dp, _i64, _c_dp, _c_dp, _i, ctypes.c_void_p]),
}

MODE_FULL, MODE_UU, MODE_PHIPHI, MODE_PHIROW = 0, 1, 2, 3
FLAG_DIRICHLET, FLAG_ACTIVE = 1, 2
LAYOUT_FULL, LAYOUT_UU, LAYOUT_PHI = 0, 1, 2
CONS_SELECT, CONS_ZERO, CONS_COPY, CONS_EXCLUDE = 0, 1, 2, 3
OPT_GENERIC_APPLY, OPT_SWEEP_ROWS, OPT_SWEEP_MIN_NSIDE, OPT_SWEEP_COLRING = 1, 2, 3, 4
CHEB_FIRST, CHEB_LAST, CHEB_NOACC = 1, 2, 4
SMOOTH_ADD_D0 = 1


def set_option(key: int, value: int):
    call("pff_set_option", key, value)


class PffError(RuntimeError):
    """A libpff_b200 entry point returned a non-zero status."""


class _Material(ctypes.Structure):
    _fields_ = [("lame_lambda", ctypes.c_double), ("mu", ctypes.c_double),
                ("g_c", ctypes.c_double), ("kappa", ctypes.c_double), ("eps", ctypes.c_double)]


_lib = None


def load(build_if_missing: bool = True):
    """Load (building first if needed) the in-tree CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing and not os.path.exists(LIB_PATH):
        from . import _build
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libpff_b200.so not found at {LIB_PATH}; run paper_2005_00331_b200._build")
    L = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.pff_abi_version() != 1:
        raise ImportError("libpff_b200.so ABI version mismatch")
    _lib = L
    return L


_fns: dict = {}


def call(name: str, *args):
    fn = _fns.get(name)
    if fn is None:
        fn = _fns[name] = getattr(load(), name)
    rc = fn(*args)
    if rc != 0:
        msg = load().pff_last_error().decode(errors="replace")
        raise PffError(f"{name} failed ({rc}): {msg}")
    return rc


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2005_00331_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle() -> int:
    """cudaStream_t of torch's current stream on the current device (the
    stream every entry point is ordered on)."""
    if _raw_stream is not None:   # the same query without torch's Python device plumbing
        return _raw_stream(torch._C._cuda_getDevice())
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def material(params) -> _Material:
    return _Material(params.lame_lambda, params.mu, params.g_c, params.kappa, params.eps)
