"""Builds libqvb.so (the C-ABI library of include/qvb.h) in-tree for sm_100a.

Every csrc/*.cu is compiled by nvcc with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false`` and
linked into paper_2305_10863_b200/libqvb.so. ``-fmad=false`` is a second line
of defence for the fp64 exactness of K1 (the kernels already use explicit
round-to-nearest intrinsics everywhere).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libqvb.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
                "-Xcompiler", "-Wall", "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "qvb.h")])


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    newest_dep = max(os.path.getmtime(p) for p in _deps() + [src])
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [NVCC, *FLAGS, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for o in glob.glob(os.path.join(OBJ, "*.o")):
            os.remove(o)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_cpp()
    return LIB


CPP_LIB = os.path.join(PKG, "libqv_b200.so")


def build_cpp() -> str:
    """libqv_b200.so: the qv:: C++ drop-in (cpp/qv_b200.cpp) over libqvb.so."""
    src = os.path.join(PKG, "cpp", "qv_b200.cpp")
    deps = [src, os.path.join(PKG, "cpp", "qv_b200.hpp"), os.path.join(ROOT, "include", "qvb.h"), LIB]
    if os.path.exists(CPP_LIB) and os.path.getmtime(CPP_LIB) >= max(os.path.getmtime(p) for p in deps):
        return CPP_LIB
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-o", CPP_LIB, src,
           "-L" + PKG, "-lqvb", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"g++ failed for the qv:: drop-in:\n{r.stdout}\n{r.stderr}")
    return CPP_LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
