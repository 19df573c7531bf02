"""ctypes binding of librevgpu.so (include/revgpu.h).

The shared library is built in-tree (`make -C paper_2003_04617_b200/csrc`,
or `__graft_entry__.build()`), statically linked against cudart, and loaded
from this package directory.  There is no fallback: if the library is
missing, or a call reports a CUDA error, `NativeLibraryError` is raised.
"""

import ctypes
import os
import threading

from .errors import NativeLibraryError

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# REVGPU_LIB: build-variant override (kernel tuning experiments only)
LIB_PATH = os.environ.get("REVGPU_LIB") or os.path.join(PKG_DIR, "librevgpu.so")
CSRC = os.path.join(PKG_DIR, "csrc")

RL_OK = 0
RL_ERR_INVALID = -1
RL_ERR_CUDA = -2
RL_ERR_NO_DEVICE = -3
ABI_VERSION = 1

_lib = None
_lock = threading.Lock()

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double
_sz = ctypes.c_size_t
_ull_p = ctypes.POINTER(ctypes.c_ulonglong)

# symbol -> (restype, argtypes); the exported surface of include/revgpu.h
SIGNATURES = {
    "rl_abi_version": (ctypes.c_int, []),
    "rl_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "rl_last_error": (ctypes.c_char_p, []),
    "rl_besselj_grad_f64": (ctypes.c_int, [_i32, _vp, _i64, _f64, _f64, _f64, _i64, _i32, _vp,
                                           _vp, _vp, _vp, _vp]),
    "rl_besselj_grad_f64_host": (ctypes.c_int, [_i32, _vp, _i64, _f64, _f64, _f64, _i64, _i32,
                                                _vp, _vp, _vp, _ull_p, _ull_p, _i32]),
    "rl_ba_jac_f64": (ctypes.c_int, [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _f64, _i32,
                                     _vp, _vp, _vp, _vp, _vp, _vp]),
    "rl_ba_jac_f64_host": (ctypes.c_int, [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _f64,
                                          _i32, _vp, _vp, _vp, _ull_p, _i32]),
    "rl_gmm_workspace_bytes": (_sz, [_i32, _i32, _i64]),
    "rl_gmm_grad_f64": (ctypes.c_int, [_i32, _i32, _i64, _i64, _vp, _vp, _vp, _vp, _f64, _i32,
                                       _f64, _f64, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "rl_gmm_grad_f64_host": (ctypes.c_int, [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _f64, _i32,
                                            _f64, _f64, _i32, _vp, _ull_p, _i32]),
    "rl_gmm_grad_shard_f64_host": (ctypes.c_int, [_i32, _i32, _i64, _i64, _vp, _vp, _vp, _vp,
                                                  _f64, _i32, _f64, _f64, _i32, _i32, _vp, _ull_p,
                                                  _i32]),
    "rl_gmm_gradient_f64": (ctypes.c_int, [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _f64, _i32,
                                           _f64, _f64, _f64, _i32, _vp, _vp, _vp, _vp, _vp, _vp,
                                           _sz, _vp]),
    "rl_gmm_run_f64": (ctypes.c_int, [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _f64, _i32, _f64,
                                      _f64, _f64, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "rl_gmm_gradient_f64_host": (ctypes.c_int, [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _f64,
                                                _i32, _f64, _f64, _f64, _i32, _vp,
                                                ctypes.POINTER(ctypes.c_double), _ull_p, _i32]),
    "rl_seq_sum_f64": (ctypes.c_int, [_vp, _i64, _f64, _i64, _i32, _vp, _vp, _vp]),
    "rl_gmm_statement_count": (ctypes.c_int64, [_i32, _i32, _i64, _i64, _i64]),
    "rl_besselj_run_f64_host": (ctypes.c_int, [_i32, _vp, _i64, _f64, _f64, _i64, _i32, _i32,
                                               _vp, _vp, _vp, _ull_p, _i32]),
    "rl_besselj_hess_f64_host": (ctypes.c_int, [_i32, _vp, _i64, _f64, _f64, _f64, _i64, _i32,
                                                _vp, _vp, _vp, _vp, _ull_p, _i32]),
    "rl_ba_residuals_f64_host": (ctypes.c_int, [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp,
                                                _f64, _i32, _vp, _vp, _ull_p, _i32]),
    "rl_gmm_run_f64_host": (ctypes.c_int, [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _f64, _i32,
                                           _f64, _f64, _f64, _i32, _i32, _vp, _ull_p, _ull_p,
                                           _i32]),
    "rl_besselj_run_f64": (ctypes.c_int, [_i32, _vp, _i64, _f64, _f64, _i64, _i32, _i32, _vp, _vp,
                                          _vp, _vp, _vp]),
    "rl_ba_residuals_f64": (ctypes.c_int, [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _f64, _i32,
                                           _vp, _vp, _vp, _vp]),
    "rl_gmm_objective_f64": (ctypes.c_int, [_i32, _i32, _i64, _i64, _vp, _vp, _vp, _vp, _f64,
                                            _i32, _f64, _f64, _i32, _i32, _vp, _vp, _vp, _vp, _sz,
                                            _vp]),
    "rl_besselj_hess_f64": (ctypes.c_int, [_i32, _vp, _i64, _f64, _f64, _f64, _i64, _i32, _vp,
                                           _vp, _vp, _vp, _vp, _vp]),
    "rl_ba_jac_csr_f64": (ctypes.c_int, [_i32, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp,
                                         _f64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rl_ba_jac_csr_f64_host": (ctypes.c_int, [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _f64,
                                              _i32, _vp, _vp, _vp, _vp, _ull_p, _i32]),
}


def lib():
    """Load (once) and return the ctypes handle; raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} is missing: build it with `make -C {CSRC}` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        try:
            handle = ctypes.CDLL(LIB_PATH)
        except OSError as err:
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {err}") from err
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        v = handle.rl_abi_version()
        if v != ABI_VERSION:
            raise NativeLibraryError(f"librevgpu ABI {v}, expected {ABI_VERSION}")
        _lib = handle
    return _lib


def check(rc, what):
    """Raise for a negative (usage / CUDA) status; return positive codes."""
    if rc < 0:
        L = lib()
        detail = L.rl_last_error().decode(errors="replace")
        raise NativeLibraryError(
            f"{what}: {L.rl_strerror(rc).decode()} ({rc}): {detail}")
    return rc


def exported_symbols():
    return list(SIGNATURES)
