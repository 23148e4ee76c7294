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


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=(), csrc: str = None) -> str:
    """Compile every csrc/*.cu into `out` (default: the in-tree libgtc.so);
    `defines` (-D flags) and another `csrc` directory only for experiment
    builds (tools/build_variant.py)."""
    srcs = sorted(glob.glob(os.path.join(csrc or os.path.join(PKG, "csrc"), "*.cu")))
    newest = max(os.path.getmtime(s) for s in sources())
    if not force and not defines and not csrc and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    nccl = _nccl_root()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc"), "-I", os.path.join(nccl, "include"),
           "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
           f"-Xlinker=-rpath={os.path.join(nccl, 'lib')}",
           *[f"-D{d}" for d in defines], "-o", out + ".tmp", *srcs]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
