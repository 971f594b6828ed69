"""Build recipe for the in-tree CUDA library (sm_100a only).

`python -m paper_2004_02297_b200._build` (or `__graft_entry__.build()`)
compiles csrc/*.cu into paper_2004_02297_b200/libadt.so with nvcc. No JIT
cache is used: the .so sits in the package directory so it travels to the
GPU box with the repository snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libadt.so")
SOURCES = [os.path.join(PKG, "csrc", "adt_kernels.cu"), os.path.join(PKG, "csrc", "adt_host.cpp")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# No --use_fast_math: subnormals and NaN payloads travel through the byte path
# untouched, and the float64 norm must not flush (SURVEY.md §7 hard part 6).
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-pthread", "-shared", "-lpthread",
              "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the ADT library needs the CUDA 12.9 toolkit to build")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = SOURCES + [os.path.join(ROOT, "include", "adt.h")] + \
        [os.path.join(PKG, "csrc", f) for f in os.listdir(os.path.join(PKG, "csrc")) if f.endswith(".cuh")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-o", tmp, *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    with open(os.path.join(PKG, "csrc", "ptxas.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stderr, file=sys.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
