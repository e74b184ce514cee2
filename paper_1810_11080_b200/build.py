"""Build the C-ABI library libhosweep_b200.so in-tree (sm_100a).

nvcc compiles the CUDA kernels for ``-gencode arch=compute_100a,code=sm_100a``
with ``-lineinfo``; g++ compiles the host setup with ``-ffp-contract=off`` (the
graph weights must be bit-identical to the reference element-wise arithmetic);
nvcc links both with a static CUDA runtime so the .so only needs libcuda at
run time.  The library lands in ``paper_1810_11080_b200/lib/`` and travels to
the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libhosweep_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES_CU = ["hsw_kernels.cu", "hsw_dmma.cu", "hsw_dmma1.cu", "hsw_dmma2.cu", "hsw_setup.cu"]
SOURCES_CPP = ["hsw_host.cpp"]
HEADERS = ["hsw_internal.hpp", os.path.join(ROOT, "include", "hosweep_b200.h")]


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose_ptxas: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    hdrs = [h if os.path.isabs(h) else os.path.join(CSRC, h) for h in HEADERS]
    objs = []
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    for s in SOURCES_CU:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, s + ".o")
        if force or _stale(obj, [src] + hdrs):
            dbg = ["-DHSW_DEBUG_BOUNDS"] if os.environ.get("HSW_DEBUG_BOUNDS") == "1" else []
            cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", *dbg,
                   "--expt-relaxed-constexpr", *inc, "-c", src, "-o", obj]
            if verbose_ptxas:
                cmd.insert(1, "-Xptxas=-v")
            _run(cmd)
        objs.append(obj)
    for s in SOURCES_CPP:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, s + ".o")
        if force or _stale(obj, [src] + hdrs):
            _run([CXX, "-O3", "-std=c++17", "-fPIC", "-ffp-contract=off", "-mavx2", "-pthread",
                  "-Wall", "-Wextra", "-Wno-unused-parameter", *inc, "-I", "/usr/local/cuda/include",
                  "-c", src, "-o", obj])
        objs.append(obj)
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs,
              "-Xcompiler", "-pthread", "-Xlinker", "--no-undefined"])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="--ptxas" in sys.argv)
