"""Build the in-tree shared library paper_2302_07499_b200/libnlfem_gpu.so.

nvcc compiles the CUDA translation unit for sm_100a only (no PTX fallback,
no other architectures) with -fmad=false so the geometric predicates keep the
reference's FMA-free rounding; the Monte Carlo stream uses
explicit fma() where it wants one.  The host setup (mesh / element table /
dof map / forcing) is compiled with g++ -ffp-contract=off for the same reason.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libnlfem_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CU_SOURCES = ["nlfem_gpu.cu", "nlfem_cg.cu", "nlfem_setup.cu", "nlfem_gpu2d.cu"]
CPP_SOURCES = ["host_setup.cpp"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-Xptxas", "-v",
]


def _run(cmd, log):
    log.write(" ".join(cmd) + "\n")
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra_flags=(), out=None) -> str:
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(INC, f) for f in os.listdir(INC)] + [__file__]
    lib = out or LIB
    if not force and not _stale(lib, deps):
        return lib
    objdir = os.path.join(HERE, "_build")
    os.makedirs(objdir, exist_ok=True)
    logpath = os.path.join(objdir, "build.log")
    objs = []
    with open(logpath, "w") as log:
        for src in CU_SOURCES:
            obj = os.path.join(objdir, src + ".o")
            _run([NVCC, *NVCC_FLAGS, *extra_flags, "-I", INC, "-I", CSRC, "-c",
                  os.path.join(CSRC, src), "-o", obj], log)
            objs.append(obj)
        for src in CPP_SOURCES:
            obj = os.path.join(objdir, src + ".o")
            _run(["g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-I", INC,
                  "-c", os.path.join(CSRC, src), "-o", obj], log)
            objs.append(obj)
        _run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib,
              *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"], log)
    if verbose:
        sys.stdout.write(open(logpath).read())
    return lib


CHECKED_LIB = os.path.join(HERE, "libnlfem_gpu_checked.so")


def build_checked(force: bool = False) -> str:
    """libnlfem_gpu_checked.so: the main translation unit with -DNLFEM_CHECKED=1
    (canaries around every device buffer, verified after each run: the memory
    checking substitute while compute-sanitizer is closed on the GPU pool),
    linked with the default build's other objects.  Used only by
    tests/test_gpu_checked.py through NLFEM_GPU_LIB."""
    build()
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(INC, f) for f in os.listdir(INC)] + [__file__]
    if not force and not _stale(CHECKED_LIB, deps):
        return CHECKED_LIB
    objdir = os.path.join(HERE, "_build")
    obj = os.path.join(objdir, "nlfem_gpu_checked.o")
    others = [os.path.join(objdir, f + ".o") for f in CU_SOURCES + CPP_SOURCES
              if f != "nlfem_gpu.cu"]
    with open(os.path.join(objdir, "build_checked.log"), "w") as log:
        _run([NVCC, *NVCC_FLAGS, "-DNLFEM_CHECKED=1", "-I", INC, "-I", CSRC, "-c",
              os.path.join(CSRC, "nlfem_gpu.cu"), "-o", obj], log)
        _run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", CHECKED_LIB,
              obj, *others, "-lcudart_static", "-lrt", "-ldl", "-lpthread"], log)
    return CHECKED_LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
