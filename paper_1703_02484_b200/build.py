"""Build libbd_b200.so (sm_100a) in-tree with nvcc.

    python -m paper_1703_02484_b200.build          # or __graft_entry__.build()

-fmad=false: the exact paths must round a*b+c twice, like the reference's
numba/numpy arithmetic; kernels that want a fused multiply-add call fma()
explicitly (bd_allpairs.cuh, FAST).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "_lib", "libbd_b200.so")
SOURCES = ["bd_capi.cu"]
HEADERS = ["bd_common.cuh", "bd_exec.cuh", "bd_step.cuh", "bd_allpairs.cuh", "bd_allpairs_fast.cuh", "bd_verlet.cuh",
           "bd_drivers.cuh", "bd_ops.cuh", "bd_allpairs_sym.cuh", "bd_build.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "--shared", "-cudart", "shared",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "bd_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile libbd_b200.so (or, with `out` / `defines`, a kernel-variant
    build of the same sources for tools/ experiments)."""
    out = out or LIB
    if out == LIB and not defines and not force and not _stale():
        return LIB
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", out, *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
