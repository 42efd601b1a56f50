"""Build libgrca.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = [os.path.join(PKG, "csrc", "grca.cu")]
DEPS = SRC + [os.path.join(PKG, "csrc", "grca_device.cuh"), os.path.join(ROOT, "include", "grca.h")]
LIB = os.path.join(PKG, "libgrca.so")

def nccl_root() -> str:
    """NCCL headers + library: the nvidia-nccl wheel torch itself loads (one libnccl.so.2 per process)."""
    import importlib

    try:
        paths = list(importlib.import_module("nvidia.nccl").__path__)
    except ImportError:
        paths = []
    for base in paths:
        if os.path.exists(os.path.join(base, "include", "nccl_device.h")):
            return base
    raise RuntimeError("NCCL >= 2.28 headers (nvidia-nccl wheel with include/nccl_device.h) not found")


NCCL = nccl_root()
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-ftz=true",
    "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared", "-I", os.path.join(ROOT, "include"),
    "-I", os.path.join(NCCL, "include"), "-L", os.path.join(NCCL, "lib"), "-l:libnccl.so.2",
    "-Xlinker", "-rpath," + os.path.join(NCCL, "lib"),
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def build_variant(out: str, defines: list) -> str:
    """A/B build (tools/ab.py): the same sources with extra -D macros, to `out`."""
    subprocess.check_call([nvcc()] + NVCC_FLAGS + [f"-D{d}" for d in defines] + SRC + ["-o", out])
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    stale = force or not os.path.exists(LIB) or any(os.path.getmtime(d) > os.path.getmtime(LIB) for d in DEPS)
    if stale:
        tmp = f"{LIB}.{os.getpid()}.tmp"
        cmd = [nvcc()] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + SRC + ["-o", tmp]
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
