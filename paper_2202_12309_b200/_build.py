"""Build libph.so in-tree: nvcc for sm_100a (no JIT cache; the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libph.so")
SOURCES = ["kernels.cu", "stage2.cu", "api.cu", "mesh.cpp"]
HEADERS = ["device.cuh", "point.cuh", "mesh.hpp", os.path.join("..", "..", "include", "ph.h")]


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


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None, extra=()) -> str:
    target = out or LIB
    if not force and not defines and out is None and not _stale():
        return LIB
    nccl = nccl_root()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", f"-I{nccl}/include",
           *[f"-D{d}" for d in defines], *extra,
           "-o", target + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES],
           f"-L{nccl}/lib", "-l:libnccl.so.2", f"-Xlinker", f"-rpath={nccl}/lib"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(target + ".tmp", target)
    return target


STRICT_LIB = os.path.join(HERE, "libph_strict.so")


def build_strict(force: bool = False) -> str:
    """Strict diagnostic build: no FMA contraction, IEEE division / square root,
    the oracle's division by dx -- run with PH_STAGE_V1=1 PH_NO_HBASE=1 so the round-1 stage kernel
    with the general finish runs; GPU fluxes then agree with the oracle's nearly bitwise."""
    if (not force and os.path.exists(STRICT_LIB) and os.path.exists(LIB)
            and os.path.getmtime(STRICT_LIB) >= os.path.getmtime(LIB) and not _stale()):
        return STRICT_LIB
    return build(force=True, defines=("PH_STRICT",), out=STRICT_LIB, extra=("-fmad=false",))


JITTER_LIB = os.path.join(HERE, "libph_jitter.so")


def build_jitter(force: bool = False) -> str:
    """Race-probe build (-DPH_JITTER=1, point.cuh): warps sleep at random probe points; its results must
    equal the normal build's bit for bit (tests/test_gpu_races.py)."""
    if (not force and os.path.exists(JITTER_LIB) and os.path.exists(LIB)
            and os.path.getmtime(JITTER_LIB) >= os.path.getmtime(LIB) and not _stale()):
        return JITTER_LIB
    return build(force=True, defines=("PH_JITTER=1",), out=JITTER_LIB)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
