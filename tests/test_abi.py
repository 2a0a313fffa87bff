"""The C-ABI library builds for sm_100a, loads without a GPU, and exports exactly the
entry points include/docthresh_b200.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_1210_3165_b200 import _lib, build

HEADER = os.path.join(ROOT, "include", "docthresh_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(dtb_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("dtb_binarize", "dtb_to_gray", "dtb_window_stats", "dtb_last_error",
                 "dtb_binarize_batch", "dtb_rgb_binarize", "dtb_sampled_stats"):
        assert name in syms


def test_library_builds_and_loads():
    path = build.build()
    assert os.path.exists(path)
    lib = _lib.lib()
    assert lib.dtb_abi_version() == 1
    assert lib.dtb_last_error() == b""


def test_library_exports_every_declared_symbol():
    build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (dtb_\w+)", out))
    assert set(declared_symbols()) <= exported
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name)


def test_python_signature_table_covers_header():
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def _header_prototypes():
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    protos = {}
    for m in re.finditer(r"^\s*(?:int|const char \*)\s*(dtb_\w+)\s*\(([^)]*)\)\s*;", text,
                         re.M | re.S):
        args = [a.strip() for a in m.group(2).split(",") if a.strip() and a.strip() != "void"]
        protos[m.group(1)] = args
    return protos


def test_python_signature_types_match_header():
    """Every ctypes argtype agrees with the C prototype (pointer / int64 / int32 / double)."""
    want = {"int64_t": ctypes.c_int64, "int32_t": ctypes.c_int32, "double": ctypes.c_double,
            "uint64_t": ctypes.c_uint64}
    protos = _header_prototypes()
    assert set(protos) == set(_lib.SIGNATURES)
    for name, args in protos.items():
        got = _lib.SIGNATURES[name]
        assert len(got) == len(args), name
        for a, t in zip(args, got):
            exp = ctypes.c_void_p if "*" in a else want[a.split()[0]]
            assert t is exp, f"{name}: {a!r} bound as {t}"


def test_library_is_sm100a():
    build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_arguments_fail_without_touching_the_device():
    lib = _lib.lib()
    rc = lib.dtb_binarize(1, 8, 8, 8, 0, 8, 0, 8, 1, 8, None, 0, 4, 2, 0.5, 128.0, None)
    assert rc == _lib.DTB_E_INVALID
    assert b"window" in lib.dtb_last_error()
    rc = lib.dtb_binarize(1, 8, 8, 8, 0, 8, 0, 8, 1, 8, None, 0, 5, 2, -0.5, 128.0, None)
    assert rc == _lib.DTB_E_INVALID and b"k_sauvola" in lib.dtb_last_error()
    rc = lib.dtb_binarize(1, 8, 8, 8, 0, 8, 0, 8, 1, 8, None, 0, 5, 1, -0.5, 0.0, None)
    assert rc == _lib.DTB_E_INVALID and b"r:" in lib.dtb_last_error()
    rc = lib.dtb_binarize(1, 8, 4, 8, 0, 16, 0, 16, 1, 8, None, 0, 5, 2, 0.5, 128.0, None)
    assert rc == _lib.DTB_E_INVALID and b"rows" in lib.dtb_last_error()
    with pytest.raises(ValueError, match="window"):
        _lib.check(lib.dtb_window_stats(1, 8, 8, 8, 2, None, None, None, None, None, None), "x")
