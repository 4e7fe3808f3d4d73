"""Build the sm_100a C-ABI library libeik.so in-tree (explicit nvcc; no JIT cache)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = [os.path.join(PKG, "csrc", "eik.cu")]
DEPS = SRC + [os.path.join(PKG, "csrc", "eik_kernels.cuh"), os.path.join(ROOT, "include", "eik.h")]
LIB = os.path.join(PKG, "libeik.so")
LIB_CHECKS = os.path.join(PKG, "libeik_checks.so")   # -DEIK_CHECKS: device bounds checks
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def _nvcc(out, extra):
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *FLAGS, *extra, "-o", tmp, *SRC])
    os.replace(tmp, out)


def build(force: bool = False, verbose: bool = False, checks: bool = True) -> str:
    if force or needs_build():
        _nvcc(LIB, ["-Xptxas", "-v"] if verbose else [])
    if checks and (force or not os.path.exists(LIB_CHECKS) or
                   os.path.getmtime(LIB_CHECKS) < os.path.getmtime(LIB)):
        _nvcc(LIB_CHECKS, ["-DEIK_CHECKS"])
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
