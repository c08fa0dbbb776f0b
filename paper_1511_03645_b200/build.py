"""Build libadjamr_b200.so in-tree with nvcc for sm_100a.

Exact-arithmetic translation units (k1_exact, k2_ghost, k3_flag) are compiled
with -fmad=false so their results are bitwise identical to the numpy
reference; the fast step kernel (k1_fast) keeps FMA contraction.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libadjamr_b200.so")
BUILD = os.path.join(HERE, "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
UNITS = {
    "abi.cu": [],
    "k1_exact.cu": ["-fmad=false"],
    "k2_ghost.cu": ["-fmad=false"],
    "k3_flag.cu": ["-fmad=false"],
    "k1_fast.cu": [],
    "k5_flagmask.cu": [],
    "host_cluster.cpp": [],
    "host_ghost.cpp": [],
}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, ptxas_info: bool = False, lib: str = LIB, build_dir: str = BUILD,
          extra: list[str] | None = None) -> str:
    """Compile every unit (only stale ones) and link ``lib``."""
    BUILD = build_dir
    LIB = lib
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, "adj_common.cuh"),
               os.path.join(HERE, "..", "include", "adjamr_b200.h")]
    objs = []
    procs = []
    for src, flags in UNITS.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o").replace(".cpp", ".o"))
        objs.append(o)
        if _stale(o, [s, *headers, __file__]):
            cmd = [nvcc(), *ARCH, *COMMON, *flags, *(extra or []), "-c", s, "-o", o]
            if ptxas_info:
                cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for cmd, pr in procs:
        out, _ = pr.communicate()
        if pr.returncode != 0:
            raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{out}")
        if out and (verbose or ptxas_info):
            print(out)
    if _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(verbose=True, ptxas_info="-v" in sys.argv)
    print(LIB)
