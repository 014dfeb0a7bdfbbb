"""Build libtsq_b200.so in-tree for sm_100a (``python -m paper_1505_00558_b200.build``).

The shared library is the product: the CUDA kernels of csrc/ behind the C
ABI declared in include/tsq.h.  It is built next to this file so it travels
with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtsq_b200.so")
TRACE_LIB = os.path.join(HERE, "libtsq_b200_trace.so")  # profiling build (-DTSQ_TRACE)
# invariant-checked build (-DTSQ_DEBUG_CHECKS, scripts/gpu_debug_checks.sh)
DEBUG_LIB = os.path.join(ROOT, "build_var", "libtsq_dbg.so")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(ROOT, "include", "tsq.h")])


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False, trace: bool = False,
          debug_checks: bool = False) -> str:
    lib = TRACE_LIB if trace else (DEBUG_LIB if debug_checks else LIB)
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    if not force and up_to_date(lib):
        return lib
    cmd = [nvcc_path(), ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-Wall", "-diag-suppress=177,1886", "-shared", "-o", lib + ".tmp",
           os.path.join(CSRC, "tsq_capi.cu")]
    if trace:
        cmd.insert(1, "-DTSQ_TRACE")
    if debug_checks:
        cmd.insert(1, "-DTSQ_DEBUG_CHECKS")
    if verbose:
        cmd.insert(5, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                trace="--trace" in sys.argv, debug_checks="--debug-checks" in sys.argv))
