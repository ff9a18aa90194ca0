"""Build libsb200.so (sm_100a) in-tree with nvcc.

    python -m paper_2009_10917_b200.build [--force] [--verbose]

The library is plain C ABI (include/sb200.h) over hand-written CUDA; cudart
is linked statically so the .so has no dependency on a particular runtime
build.  -fmad=false is belt and braces: the kernels use __dmul_rn/__dadd_rn
explicitly, which are never contracted to FMA.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libsb200.so")
HEADER = os.path.join(ROOT, "include", "sb200.h")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-O2",
         "--expt-relaxed-constexpr"]


def nccl_include() -> str:
    """NCCL >= 2.28 headers (nccl_device.h) from the nvidia-nccl wheel torch uses;
    /usr/include/nccl.h is an older release without the device API."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    roots = list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []
    for r in roots:
        inc = os.path.join(r, "include")
        if os.path.exists(os.path.join(inc, "nccl_device.h")):
            return inc
    raise RuntimeError("nccl_device.h (NCCL >= 2.28 headers) not found in the nvidia-nccl package")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [HEADER]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-I" + nccl_include(), "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = LIB + ".tmp"
    subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static", "-ldl"], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
