"""Builds paper_2511_12235_b200/libctsm_b200.so with nvcc for sm_100a.

csr.cu, weights.cu and line.cu (bit-exact CSR emission and weight API) are compiled with -fmad=false so that no FMA
contraction changes the reference's rounding; the
matrix-free kernels (mf.cu) keep contraction on.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libctsm_b200.so")
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
          "-I" + CSRC, "-I" + os.path.join(HERE, "..", "include")] + ARCH
# tuning experiments only (tools/sweep3d.sh): extra nvcc flags, e.g. -DCTSM_KZCS=4
COMMON += os.environ.get("CTSM_NVCC_EXTRA", "").split()
UNITS = {
    "csr.cu": ["-fmad=false"],
    "line.cu": ["-fmad=false"],
    "weights.cu": ["-fmad=false"],
    "oracles.cu": ["-fmad=false"],
    "mf.cu": [],
    "solver.cu": ["-fmad=false"],
    "capi.cu": [],
    "io.cu": [],
    "api.cpp": [],
    "multi.cu": [],
}


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(HERE, "..", "include", "ctsm_b200.h"))
    headers.append(os.path.join(HERE, "..", "include", "ctsm_b200", "ctsm.hpp"))
    objs = []
    for unit, extra in UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(OBJ, os.path.splitext(unit)[0] + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [NVCC, "-c", src, "-o", obj] + COMMON + extra
            if verbose:
                cmd += ["-Xptxas", "-v"]
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        cmd = [NVCC, "-shared", "-o", LIB] + objs + ARCH + ["-lcudart", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
