"""Build libcbp.so (the C-ABI library of include/cbp.h) in-tree with nvcc for
sm_100a.  Run as ``python -m paper_1907_10526_b200.build`` or via
``__graft_entry__.build()``."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libcbp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
    "-I", CSRC,
]


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cuh", ".h")))


def build_debug() -> str:
    """libcbp_debug.so: the same library with device-side index checks (CBP_DEBUG_CHECKS)."""
    out = os.path.join(PKG, "libcbp_debug.so")
    cmd = [NVCC, *NVCC_FLAGS, "-DCBP_DEBUG_CHECKS", "-o", out, os.path.join(CSRC, "cbp.cu")]
    subprocess.run(cmd, check=True, capture_output=True)
    return out


def build_variant(out: str, defines: list[str]) -> str:
    """an A/B build of the same sources with extra -D macros (tools/ab_time.py)"""
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", out, os.path.join(CSRC, "cbp.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(res.stderr[-3000:])
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    deps = sources() + [os.path.join(ROOT, "include", "cbp.h"), os.path.abspath(__file__)]
    stale = (not os.path.exists(LIB)) or any(os.path.getmtime(d) > os.path.getmtime(LIB)
                                             for d in deps)
    if not (force or stale):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *NVCC_FLAGS, "-o", tmp, os.path.join(CSRC, "cbp.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "build_ptxas.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
