"""Build libhelinear.so in-tree (sm_100a CUDA kernels + host C++), no torch extension machinery.

    python -m paper_2305_18396_b200.build            # incremental
    python -m paper_2305_18396_b200.build --force

nvcc cross-compiles sm_100a on a machine without a GPU; the .so lands in
paper_2305_18396_b200/lib/ and travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(LIBDIR, "libhelinear.so")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp",
                     "-I" + os.path.join(ROOT, "include")] + os.environ.get("HELINEAR_NVCC_EXTRA", "").split()
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-fopenmp", "-Wall", "-Wno-unknown-pragmas", "-I" + os.path.join(CUDA_HOME, "include"),
             "-I" + os.path.join(ROOT, "include")]

CU_SOURCES = ["kernels.cu"]
CXX_SOURCES = ["ctx.cpp", "client.cpp"]
# every header under csrc/ (and include/helinear.h): an edit to any of them rebuilds every object
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".h", ".cuh")))


def _newer(src_list, target) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "helinear.h")]
    objs = []
    for src in CU_SOURCES + CXX_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJDIR, src + ".o")
        objs.append(o)
        if force or _newer([s] + hdrs, o):
            if src.endswith(".cu"):
                cmd = [NVCC] + NVCC_FLAGS + ["-c", s, "-o", o]
            else:
                cmd = ["g++"] + CXX_FLAGS + ["-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
    if force or _newer(objs, LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lquadmath", "-lgomp", "-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
