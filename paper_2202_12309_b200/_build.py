"""Build libph.so in-tree: nvcc for sm_100a (no JIT cache; the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libph.so")
SOURCES = ["kernels.cu", "api.cu", "mesh.cpp"]
HEADERS = ["device.cuh", "mesh.hpp", os.path.join("..", "..", "include", "ph.h")]


def nccl_root() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        return list(spec.submodule_search_locations)[0]
    return "/usr"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    return any(os.path.getmtime(f) > t for f in files if os.path.exists(f))


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    target = out or LIB
    if not force and not defines and out is None and not _stale():
        return LIB
    nccl = nccl_root()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", f"-I{nccl}/include",
           *[f"-D{d}" for d in defines],
           "-o", target + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES],
           f"-L{nccl}/lib", "-l:libnccl.so.2", f"-Xlinker", f"-rpath={nccl}/lib"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
