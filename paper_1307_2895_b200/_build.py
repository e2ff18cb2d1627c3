"""In-tree build of the sm_100a library ``libhifde_gpu.so``.

nvcc cross-compiles for B200 (``-gencode arch=compute_100a,code=sm_100a``) on
a machine without a GPU; the CUDA runtime is linked statically so the library
loads anywhere the CUDA driver is present (and can be dlopen'ed for symbol
checks where it is not).
"""

from __future__ import annotations

import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libhifde_gpu.so")
SOURCES = [
    "csrc/kernels_factor.cu",
    "csrc/kernels_big.cu",
    "csrc/kernels_skelbig.cu",
    "csrc/kernels_solve.cu",
    "csrc/kernels_krylov.cu",
    "csrc/symbolic.cu",
    "csrc/runtime.cu",
    "csrc/comm.cu",
    "csrc/partition.cpp",
    "csrc/shard.cpp",
    "csrc/hostprof.cpp",
]
HEADERS = ["csrc/keys.h", "csrc/hifde_internal.h", "csrc/partition.h", "csrc/hostprof.h", "csrc/comm.h", "csrc/shard.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build the sm_100a library")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(PKG, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "hifde_gpu.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [_nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O3,-fopenmp,-g", "-lgomp", "-ldl",
           "-shared", "-cudart", "static", "--threads", "4",
           "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp",
           *[os.path.join(PKG, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=PKG)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force=True))
