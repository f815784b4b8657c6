"""In-tree build of libmine_b200.so (sm_100a) -- no JIT cache, so the built
library travels to the GPU box with the repo snapshot.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false  (kernels)
    g++  -O2 -ffp-contract=off                                              (host runtime)
    nvcc -shared -cudart static                                             (link)

-fmad=false / -ffp-contract=off: no FMA contraction anywhere, matching the
reference's x86-64 build bit for bit.
"""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libmine_b200.so")
PROBES = os.path.join(PKG, "libmine_b200_probes.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_INC = "/usr/local/cuda/include"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

KERNEL_SRCS = ["mine_kernels.cu", "mine_general.cu", "pearson.cu", "format.cu"]
HOST_SRCS = ["engine.cpp", "records.cpp"]
HEADERS = ["mine_kernels.h", "device_common.cuh", os.path.join("..", "..", "include", "mine_b200.h")]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def _run(cmd: list[str]) -> None:
    subprocess.run(cmd, check=True)


CHECKED_LIB = os.path.join(PKG, "libmine_b200_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """checked=True: the bounds-checked variant (device asserts, -DMB_BOUNDS_CHECK)
    as libmine_b200_checked.so, objects under build/checked (load it with
    MINE_B200_LIB); the substitute for compute-sanitizer, closed on the pool."""
    if checked:
        return _build_into(os.path.join(BUILD, "checked"), CHECKED_LIB, ["-DMB_BOUNDS_CHECK"], force, verbose)
    return _build_into(BUILD, LIB, [], force, verbose, probes=True)


def _build_into(BUILD: str, LIB: str, defs: list, force: bool, verbose: bool, probes: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.normpath(os.path.join(CSRC, h)) for h in HEADERS]
    objs = []
    for src in KERNEL_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or not _newer(o, [s] + hdrs):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17", *defs,
                   "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            _run(cmd)
        objs.append(o)
    for src in HOST_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or not _newer(o, [s] + hdrs):
            _run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-Wall", "-Wextra",
                  "-I", os.path.join(ROOT, "include"), "-I", CUDA_INC, "-c", s, "-o", o])
        objs.append(o)
    if force or not _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread", "-ldl"])
    probe_src = os.path.join(CSRC, "probes.cu")
    if probes and (force or not _newer(PROBES, [probe_src] + [os.path.normpath(os.path.join(CSRC, h)) for h in HEADERS])):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "-cudart", "static", "-o", PROBES, probe_src])
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
