"""Build librkc.so in-tree with nvcc for sm_100a (no GPU needed to compile)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(CSRC, f) for f in ("rkc_step_small_o64.cu", "rkc_step_small_o128.cu",
                                           "rkc_step_big_o64.cu", "rkc_step_big_o128.cu",
                                           "rkc_abi.cu", "rkc_conformance.cu")]
HEADERS = [os.path.join(CSRC, f) for f in ("rkc_internal.cuh", "rkc_step_impl.cuh")] + \
    [os.path.join(ROOT, "include", "rkc.h")]
LIB = os.path.join(HERE, "librkc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-shared", "-cudart", "shared"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple[str, ...] = ()) -> str:
    """Compile librkc.so; `out` / `defines` build an experiment variant beside it."""
    lib = out or LIB
    if not force and out is None and not stale():
        return LIB
    extra = os.environ.get("RKC_NVCC_EXTRA", "").split() + [f"-D{d}" for d in defines]
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), *SOURCES, "-o", lib]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return lib


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
