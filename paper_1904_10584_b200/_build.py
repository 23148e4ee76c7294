"""Build libgtc.so in-tree for sm_100a with nvcc (no JIT cache, no torch
extension machinery: the library has a plain C ABI, include/gtc.h)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libgtc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_root() -> str:
    import nvidia.nccl  # the NCCL torch loads (2.28.x); link the same copy

    return list(nvidia.nccl.__path__)[0]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu"))) + sorted(
        glob.glob(os.path.join(PKG, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "gtc.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
    newest = max(os.path.getmtime(s) for s in sources())
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    nccl = _nccl_root()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include"),
           "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
           f"-Xlinker=-rpath={os.path.join(nccl, 'lib')}",
           "-o", LIB + ".tmp", *srcs]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
