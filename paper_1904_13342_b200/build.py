"""Build libtomograd_b200.so in-tree (sm_100a).

    python -m paper_1904_13342_b200.build [-v] [--force]

CUDA sources are compiled with nvcc for ``-gencode arch=compute_100a,code=sm_100a``
with ``-lineinfo``; the host geometry (which must be bit-exact with the
reference) is compiled with the system g++ at -O2 with ``-ffp-contract=off``
and no ``-march`` (no FMA), like the reference's Release build.  Objects go to
``build/`` and the shared library next to this file, so it travels to the GPU
box with the repo snapshot.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libtomograd_b200.so")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
HOST_CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"

CU_SOURCES = ["runtime.cu", "cone.cu", "filter.cu", "planar.cu", "phantom.cu", "iterative.cu", "graph.cu"]
CPP_SOURCES = ["host_geometry.cpp"]
HEADERS = ["tg_internal.h", "device_common.cuh", "cone_kernels.cuh", "cone_fp_slab.cuh", "filter.cuh", "fft16.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-ccbin", HOST_CXX,
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
]
CXX_FLAGS = ["-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math"]


def _deps_mtime() -> float:
    files = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "tomograd_b200.h"),
                                                         __file__]
    return max(os.path.getmtime(f) for f in files if os.path.exists(f))


def _stale(src: str, obj: str, dep_mtime: float) -> bool:
    if not os.path.exists(obj):
        return True
    m = os.path.getmtime(obj)
    return m < os.path.getmtime(src) or m < dep_mtime


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def build(verbose: bool = False, force: bool = False) -> str:
    """Compile every source for sm_100a and link the C-ABI library."""
    os.makedirs(OBJ, exist_ok=True)
    dep = _deps_mtime()
    jobs = []
    vis: list = []
    for s in CU_SOURCES:
        src, obj = os.path.join(CSRC, s), os.path.join(OBJ, s + ".o")
        if force or _stale(src, obj, dep):
            jobs.append([NVCC, *NVCC_FLAGS, *vis, f"-I{INCLUDE}", f"-I{CSRC}", "-c", src, "-o", obj])
    for s in CPP_SOURCES:
        src, obj = os.path.join(CSRC, s), os.path.join(OBJ, s + ".o")
        if force or _stale(src, obj, dep):
            jobs.append([HOST_CXX, *CXX_FLAGS, *vis, f"-I{INCLUDE}", f"-I{CSRC}",
                         f"-I{CUDA_HOME}/include", "-c", src, "-o", obj])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            list(ex.map(lambda c: _run(c, verbose), jobs))
    objs = [os.path.join(OBJ, s + ".o") for s in CU_SOURCES + CPP_SOURCES]
    if jobs or force or not os.path.exists(LIB) or any(
            os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        tmp = LIB + ".tmp"
        _run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-ccbin", HOST_CXX,
              "-o", tmp, *objs, "-cudart", "static", "-Xlinker", "--exclude-libs,ALL"], verbose)
        shutil.move(tmp, LIB)
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build(a.verbose, a.force))


if __name__ == "__main__":
    main()
