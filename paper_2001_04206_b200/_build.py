"""Build recipe for the native library (sm_100a only).

    python -m paper_2001_04206_b200._build

compiles csrc/abi.cu (+ the header-only kernels) with nvcc into
``paper_2001_04206_b200/lib/liblane_b200.so`` (in-tree, so it travels to the
GPU box with the repo snapshot), and the C++ facade test driver.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "liblane_b200.so")
CLI = os.path.join(LIBDIR, "lane-bench")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off",
         "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "--expt-relaxed-constexpr"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(ROOT, "include", "lane_b200.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build_cli(force: bool = False) -> str:
    """lane-bench for the B200 path (csrc/lane_bench.cpp over the C++ facade)."""
    src = os.path.join(CSRC, "lane_bench.cpp")
    deps = [src, LIB, os.path.join(ROOT, "include", "lane_b200", "lane.hpp")]
    if not force and os.path.exists(CLI) and all(os.path.getmtime(p) <= os.path.getmtime(CLI) for p in deps):
        return CLI
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), src, "-o", CLI + ".tmp",
                    "-L", LIBDIR, "-llane_b200", "-Wl,-rpath,$ORIGIN"], check=True)
    os.replace(CLI + ".tmp", CLI)
    return CLI


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and not needs_build():
        build_cli()
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, *FLAGS, "-I", os.path.join(ROOT, "include"), "-o", tmp,
           os.path.join(CSRC, "abi.cu"), "-lnccl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    build_cli(force=True)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
