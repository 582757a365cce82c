"""Builds libl1rxg.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_1907_00463_b200.build [--verbose]

Output: paper_1907_00463_b200/_lib/libl1rxg.so (git-ignored; it travels to
the GPU box with the gpurun snapshot).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
SO = os.path.join(LIBDIR, "libl1rxg.so")
SOURCES = [os.path.join(CSRC, "l1rxg.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cuh", ".h"))] + [
    os.path.join(ROOT, "include", "l1rxg.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_cmd(verbose: bool = False) -> list:
    cmd = [NVCC, "-O3", "-lineinfo", "-std=c++17", *ARCH, "-Xcompiler", "-fPIC,-O2", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-o", SO, *SOURCES, "-lcudart", "-lcublas"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    return cmd


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    if force or not up_to_date():
        r = subprocess.run(nvcc_cmd(verbose), capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libl1rxg.so")
        if verbose:
            sys.stderr.write(r.stderr)
    return SO


if __name__ == "__main__":
    build(force=True, verbose="--verbose" in sys.argv)
    print(SO)
