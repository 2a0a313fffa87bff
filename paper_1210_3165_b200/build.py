"""Build libdocthresh_b200.so in-tree with nvcc for sm_100a (no torch JIT cache)."""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
# DTB_LIB_OUT: build a variant (e.g. the DTB_DEBUG_BOUNDS / DTB_PERTURB safety build) elsewhere;
# _lib.py loads it when DTB_LIB_PATH points at it
LIB = os.environ.get("DTB_LIB_OUT") or os.path.join(HERE, "libdocthresh_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
EXTRA = os.environ.get("DTB_NVCC_EXTRA", "").split()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


CSRC = os.environ.get("DTB_CSRC_DIR") or os.path.join(HERE, "csrc")  # A/B builds of other sources


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "docthresh_b200.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu to an object in parallel (one nvcc per file), then link."""
    if not force and up_to_date():
        return LIB
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    compile_flags = [f for f in FLAGS if f != "-shared"]
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    with tempfile.TemporaryDirectory() as td:
        objs = [os.path.join(td, os.path.basename(src) + ".o") for src in sources()]

        def compile_one(pair):
            src, obj = pair
            return subprocess.run([NVCC, *compile_flags, *EXTRA, *inc, "-c", "-o", obj, src],
                                  capture_output=True, text=True)

        with ThreadPoolExecutor(max_workers=max(1, min(len(objs), os.cpu_count() or 1))) as ex:
            results = list(ex.map(compile_one, zip(sources(), objs)))
        log = "".join(r.stdout + r.stderr for r in results)
        if any(r.returncode != 0 for r in results):
            sys.stderr.write(log)
            raise RuntimeError("nvcc build of libdocthresh_b200.so failed")
        link = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                               "-Xcompiler", "-fPIC", "-o", LIB + ".tmp", *objs],
                              capture_output=True, text=True)
        if link.returncode != 0:
            sys.stderr.write(link.stdout + link.stderr)
            raise RuntimeError("link of libdocthresh_b200.so failed")
        os.replace(LIB + ".tmp", LIB)  # atomic: a concurrent loader never sees a partial file
    if verbose:
        sys.stderr.write(log)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
