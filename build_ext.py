"""Builds libmpap.so in-tree for sm_100a (explicit nvcc; no JIT cache).

    python build_ext.py [--force]

Flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo, --fmad=false
(no FMA contraction: DESIGN.md §3 numeric contract N2), no fast-math, static
cudart (independent of the torch-bundled runtime version).
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1705_02408_b200")
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libmpap.so")
SOURCES = ["capi.cu", "build_kernels.cu", "search_kernels.cu", "mc_kernels.cu", "peak_kernels.cu", "rowshard.cu"]
HEADERS = [os.path.join(CSRC, "mpap_internal.cuh"), os.path.join(CSRC, "traj.cuh"), os.path.join(INCLUDE, "mpap.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
EXTRA = os.environ.get("MPAP_NVCC_EXTRA", "").split()   # tuning experiments only
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "-I", INCLUDE, "-I", CSRC]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + HEADERS + [__file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str = None) -> str:
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *NVFLAGS, *EXTRA, "-c", src, "-o", obj]
        out = subprocess.run(cmd, capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{out.stderr}")
        if verbose:
            sys.stderr.write(out.stderr)
        with open(os.path.join(objdir, s + ".ptxas.txt"), "w") as f:
            f.write(out.stderr)
        objs.append(obj)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{out.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    outp = None
    if "--out" in sys.argv:
        outp = sys.argv[sys.argv.index("--out") + 1]
    print(build(force="--force" in sys.argv or outp is not None, verbose=True, out=outp))
