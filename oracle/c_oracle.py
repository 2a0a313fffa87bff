"""ctypes front-end for oracle/liboracle.so (test infrastructure only)."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

METHOD_NIBLACK = 1
METHOD_SAUVOLA = 2

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "oracle.c"))):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    lib.oracle_to_gray.argtypes = [_u8p, ctypes.c_int64, _u8p]
    lib.oracle_to_gray.restype = None
    lib.oracle_run.argtypes = [_u8p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, ctypes.c_double, ctypes.c_double, _i64p, _i64p,
                               _i32p, _f64p, _f64p, _f64p, _u8p, ctypes.c_int]
    lib.oracle_run.restype = ctypes.c_int
    _lib = lib
    return lib


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _method_code(method: str) -> int:
    return {"sauvola": METHOD_SAUVOLA, "niblack": METHOD_NIBLACK}[method]


def _run(img, win, method=0, k=0.0, r=1.0, want=(), threads=1):
    img = np.ascontiguousarray(img, dtype=np.uint8)
    if img.ndim != 2:
        raise ValueError("oracle expects a 2-D uint8 image")
    h, w = img.shape
    out = {}
    for name, dt in (("S", np.int64), ("Q", np.int64), ("n", np.int32), ("mean", np.float64),
                     ("std", np.float64), ("tmap", np.float64), ("binary", np.uint8)):
        out[name] = np.empty((h, w), dtype=dt) if name in want else None
    rc = load().oracle_run(
        _ptr(img, _u8p), w, h, w, int(win), int(method), float(k), float(r),
        _ptr(out["S"], _i64p), _ptr(out["Q"], _i64p), _ptr(out["n"], _i32p),
        _ptr(out["mean"], _f64p), _ptr(out["std"], _f64p), _ptr(out["tmap"], _f64p),
        _ptr(out["binary"], _u8p), int(threads))
    if rc != 0:
        raise RuntimeError(f"oracle_run failed ({rc})")
    return out


def window_sums(img, win, threads=1):
    """(S, Q, n): exact clipped-window sums of f and f^2 and the in-bounds count."""
    o = _run(img, win, want=("S", "Q", "n"), threads=threads)
    return o["S"], o["Q"], o["n"]


def mean_std(img, win, threads=1):
    """(mean, std, count) exactly as stats.mean_std_integral returns them."""
    o = _run(img, win, want=("mean", "std", "n"), threads=threads)
    return o["mean"], o["std"], o["n"].astype(np.int64)


def binarize(img, win, method, k, r=128.0, tmap=True, threads=1):
    """(binary, tmap-or-None) exactly as threshold.binarize(engine='integral')."""
    want = ("binary", "tmap") if tmap else ("binary",)
    o = _run(img, win, _method_code(method), k, r, want=want, threads=threads)
    return o["binary"], o["tmap"]


def to_gray(rgb):
    rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
    if rgb.ndim != 3 or rgb.shape[2] != 3:
        raise ValueError(f"expected an (H, W, 3) RGB array, got shape {rgb.shape}")
    out = np.empty(rgb.shape[:2], dtype=np.uint8)
    load().oracle_to_gray(_ptr(rgb, _u8p), out.size, _ptr(out, _u8p))
    return out
