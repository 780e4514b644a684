"""Build libaxonn.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python paper_2502_08145_b200/build.py      (or __graft_entry__.build())

Objects go to paper_2502_08145_b200/build/, the library to
paper_2502_08145_b200/libaxonn.so (git-ignored, travels with gpurun).
NCCL headers and libnccl.so.2 come from the pip wheel torch itself loads
(2.28.x), so both use one NCCL instance.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libaxonn.so")
SOURCES = ["gemm_tc.cu", "gemm_simt.cu", "sym.cu", "perf_model.cpp", "axonn.cpp", "loopback.cpp", "act.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("pip NCCL (nvidia/nccl) not found")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nd = nccl_dir()
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(nd, "include")]
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-Wall", "--expt-relaxed-constexpr"]
    objs = []
    newest = 0.0
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "axonn.h")]
    dep_t = max(os.path.getmtime(d) for d in deps)
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or not os.path.exists(o) or os.path.getmtime(o) < dep_t:
            _run([nvcc()] + ARCH + flags + inc + ["-c", s, "-o", o], verbose)
        objs.append(o)
        newest = max(newest, os.path.getmtime(o))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        libdir = os.path.join(nd, "lib")
        _run([nvcc()] + ARCH + ["-shared", "-o", LIB] + objs +
             ["-L", libdir, "-l:libnccl.so.2", f"-Xlinker=-rpath,{libdir}"], verbose)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
