"""Build libcem.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libcem.so")
SOURCES = ["cem_mesh.cpp", "cem_plan.cpp", "cem_part.cpp", "cem_hex_mesh.cpp", "cem_kernels.cu", "cem_dist.cu", "cem_hex.cu",
           "cem_api.cu"]
HEADERS = ["cem_internal.h", "cem_part.h", "cem_dist.h", os.path.join("..", "..", "include", "cem.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # bitwise contract: no FMA contraction on device or host
    "--fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math,-fopenmp,-fvisibility=hidden",
    "-cudart", "static",
]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(f) > t for f in files)


def build(force: bool = False, verbose: bool = False, out: str = SO, defines=(), device_fma: bool = False) -> str:
    """device_fma: the "fast build" of SURVEY.md §8(c) -- FMA contraction in device code only (the host
    preprocessing keeps -ffp-contract=off, so geometry and masses stay the oracle's); results then
    meet the north star's tolerance instead of bit equality (tests/test_gpu_fast_build.py)."""
    if not force and out == SO and not _stale():
        return SO
    flags = [f for f in NVCC_FLAGS if not (device_fma and f == "--fmad=false")]
    if device_fma:
        flags.append("--fmad=true")
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *flags, *[f"-D{x}" for x in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose and src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = out + ".tmp"
    subprocess.check_call([NVCC, *flags, "-shared", "-o", tmp, *objs, "-lgomp", "-ldl"])
    os.replace(tmp, out)
    for o in objs:
        os.remove(o)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
