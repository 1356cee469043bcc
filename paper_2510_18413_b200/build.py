"""In-tree build of the sm_100a library and the C++ facade (no JIT cache).

libadamas_b200.so     C ABI (include/adamas_b200.h) + kernels, nvcc for sm_100a
libadamas_facade.so   C++ facade mirroring the reference operator API
                      (namespace adamas::gpu), linked against the C ABI
facade_tests          C++ parity driver for the facade (tests/cpp/)
"""
from __future__ import annotations

import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libadamas_b200.so")
DIAG_LIB = os.path.join(PKG, "libadamas_b200_diag.so")  # phase stamps compiled in (tools/phase_profile.py)
FACADE = os.path.join(PKG, "libadamas_facade.so")
FACADE_TESTS = os.path.join(ROOT, "tests", "cpp", "facade_tests")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
CUDA_HOME = os.path.dirname(os.path.dirname(os.path.realpath(NVCC)))
CUDA_INC = os.path.join(CUDA_HOME, "include")
CUDA_LIB = os.path.join(CUDA_HOME, "lib64")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-diag-suppress", "497"]


def _sources(d, exts):
    out = []
    for name in sorted(os.listdir(d)):
        if os.path.splitext(name)[1] in exts:
            out.append(os.path.join(d, name))
    return out


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(x) > t for x in deps)


def build(force: bool = False, verbose: bool = False) -> None:
    deps = _sources(CSRC, {".cu", ".cuh", ".h"}) + [os.path.join(ROOT, "include", "adamas_b200.h")]
    if force or _stale(LIB, deps):
        cmd = [NVCC, *ARCH, *NVFLAGS, "-shared", "-o", LIB, os.path.join(CSRC, "adamas_b200.cu")]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    fdir = os.path.join(CSRC, "facade")
    fdeps = _sources(fdir, {".cpp", ".hpp"}) + [LIB]
    if force or _stale(FACADE, fdeps):
        cmd = ["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
               "-I", fdir, "-I", CUDA_INC, "-o", FACADE, os.path.join(fdir, "adamas_gpu.cpp"),
               "-L", PKG, "-ladamas_b200", "-L", CUDA_LIB, "-lcudart", "-Wl,-rpath,$ORIGIN",
               f"-Wl,-rpath,{CUDA_LIB}"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    tsrc = os.path.join(ROOT, "tests", "cpp", "facade_tests.cpp")
    if os.path.exists(tsrc) and (force or _stale(FACADE_TESTS, [tsrc, FACADE])):
        cmd = ["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"), "-I", fdir,
               "-I", CUDA_INC, "-I", os.path.join(ROOT, "oracle"), "-o", FACADE_TESTS, tsrc,
               "-L", PKG, "-ladamas_facade", "-ladamas_b200", "-Wl,-rpath,$ORIGIN/../../paper_2510_18413_b200",
               "-L", os.path.join(ROOT, "oracle"), "-loracle", "-Wl,-rpath,$ORIGIN/../../oracle",
               "-L", CUDA_LIB, "-lcudart", f"-Wl,-rpath,{CUDA_LIB}"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)


def build_diag(verbose: bool = False) -> str:
    """The same library with the diagnostics compiled in (ADAMAS_DIAG=1):
    phase stamps (adamas_debug_trace) and the ADAMAS_DBG timing switches. Not
    the product: the production build leaves them out (2 % faster at config 1)."""
    cmd = [NVCC, *ARCH, *NVFLAGS, "-DADAMAS_DIAG=1", "-shared", "-o", DIAG_LIB, os.path.join(CSRC, "adamas_b200.cu")]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return DIAG_LIB


if __name__ == "__main__":
    import sys

    if "--diag" in sys.argv:
        build_diag(verbose=True)
    else:
        build(force=True, verbose=True)
