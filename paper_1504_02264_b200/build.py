"""Build the in-tree CUDA library liblesb200.so for sm_100a with nvcc.

-fmad=false and IEEE division/square root (nvcc defaults, no fast-math)
are part of the parity contract: every float op rounds once, as numpy does.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "liblesb200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo",
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC,-O2", "-shared",
    "-Xptxas", "-v",
]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(PKG, "csrc", "*.h")) + glob.glob(
        os.path.join(PKG, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "les_b200.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def nccl_flags():
    """Link the NCCL that torch itself loads (the nvidia-nccl wheel, 2.28.x,
    with an rpath to it): a process that imports torch and this library then
    has one libnccl.so.2, whichever of the two is loaded first.  Falls back
    to the system NCCL when the wheel is absent."""
    try:
        import importlib.util

        spec = importlib.util.find_spec("nvidia.nccl")
        for d in (spec.submodule_search_locations or []) if spec else []:
            lib, inc = os.path.join(d, "lib"), os.path.join(d, "include")
            if os.path.exists(os.path.join(lib, "libnccl.so.2")) and os.path.exists(os.path.join(inc, "nccl.h")):
                return ["-I", inc], ["-L", lib, "-Xlinker", "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]
    except Exception:  # noqa: BLE001
        pass
    return [], ["-lnccl"]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    nccl_inc, nccl_lib = nccl_flags()
    cmd = [NVCC, *FLAGS, "-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc"), *nccl_inc,
           "-o", LIB + ".tmp", *sources(), *nccl_lib]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building liblesb200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
