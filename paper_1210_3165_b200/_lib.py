"""ctypes binding of libdocthresh_b200.so (the C ABI in include/docthresh_b200.h).

There is no CPU fallback anywhere in this package: if the shared library is
missing or no CUDA device is visible, calls raise immediately.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DTB_LIB_PATH") or os.path.join(HERE, "libdocthresh_b200.so")  # safety builds

DTB_METHOD_NIBLACK = 1
DTB_METHOD_SAUVOLA = 2
DTB_OK = 0
DTB_E_INVALID = -1
DTB_E_CUDA = -2
DTB_E_UNSUPPORTED = -3

_c_i32, _c_i64, _c_f64, _c_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
_c_u64 = ctypes.c_uint64

# name -> argtypes, mirroring include/docthresh_b200.h one for one.
SIGNATURES = {
    "dtb_abi_version": [],
    "dtb_last_error": [],
    "dtb_to_gray": [_c_p, _c_i64, _c_p, _c_i64, _c_i32, _c_i32, _c_p],
    "dtb_binarize": [_c_p, _c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_p,
                     _c_i64, _c_p, _c_i64, _c_i32, _c_i32, _c_f64, _c_f64, _c_p],
    "dtb_binarize_batch": [_c_p, _c_i64, _c_i32, _c_i32, _c_i32, _c_p, _c_i64, _c_i32, _c_i32,
                           _c_f64, _c_f64, _c_p],
    "dtb_rgb_binarize": [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_i64, _c_p, _c_i64, _c_i32,
                         _c_i32, _c_f64, _c_f64, _c_p],
    "dtb_window_stats": [_c_p, _c_i64, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_p,
                         _c_p],
    "dtb_sampled_stats": [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_i32, _c_p, _c_p, _c_p, _c_p,
                          _c_p, _c_i32, _c_f64, _c_f64, _c_p],
    "dtb_histogram": [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p],
    "dtb_integral_tables": [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p],
    "dtb_apply_global": [_c_p, _c_i64, _c_i32, _c_i32, _c_i32, _c_p, _c_i64, _c_p],
    "dtb_gs_stats": [_c_p, _c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_p, _c_p, _c_i64,
                     _c_p, _c_i32, _c_f64, _c_f64, _c_p],
    "dtb_otsu": [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p],
    "dtb_apply_global_dev": [_c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_i64, _c_p, _c_p],
    "dtb_binarize_segments": [_c_p, _c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32,
                              _c_p, _c_i64, _c_i32, _c_i32, _c_f64, _c_f64, _c_p],
    "dtb_ipc_export": [_c_p, _c_p, _c_p],
    "dtb_ipc_import": [_c_p, _c_p],
    "dtb_ipc_close": [_c_p],
    "dtb_gs_band": [_c_p, _c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32,
                    _c_p, _c_i64, _c_i32, _c_f64, _c_f64, _c_p],
    "dtb_set_fp32_audit": [_c_p],
    "dtb_last_kernel": [],
    "dtb_debug_bb_exact": [_c_p, _c_i32],
    "dtb_debug_bb_times": [_c_p, _c_i32],
    "dtb_debug_sqrt_selftest": [_c_u64, _c_u64, _c_p],
    "dtb_confusion": [_c_p, _c_i64, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p],
    "dtb_sweep_counts": [_c_p, _c_i64, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_i64, _c_p,
                         _c_i32, _c_i32, _c_f64, _c_p, _c_p],
}

_lib = None


class NativeLibraryError(RuntimeError):
    """libdocthresh_b200.so is missing or unusable (there is no CPU fallback)."""


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} is not built; run `python -m paper_1210_3165_b200.build` "
            "(or __graft_entry__.build()). There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    allow_missing = os.environ.get("DTB_AB_ALLOW_MISSING") == "1"  # A/B builds of older sources
    for name, argtypes in SIGNATURES.items():
        if allow_missing and not hasattr(L, name):
            continue
        fn = getattr(L, name)
        fn.argtypes = argtypes
        fn.restype = (ctypes.c_char_p if name in ("dtb_last_error", "dtb_last_kernel")
                      else ctypes.c_int)
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc == DTB_OK:
        return
    msg = lib().dtb_last_error().decode(errors="replace")
    if rc == DTB_E_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"{what}: {msg} (code {rc})")
