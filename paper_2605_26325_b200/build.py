"""Builds libdare_b200.so in-tree with nvcc for sm_100a.

Kept dependency-free (no torch.utils.cpp_extension): the library is a plain
C-ABI shared object loaded with ctypes, so it can be bound from any host
language.  Flags:
  -gencode arch=compute_100a,code=sm_100a   B200 only
  -fmad=false                               never contract a*b+c (the reference
                                            never does; parity is bit-exact)
  -lineinfo                                 ncu source attribution
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdare_b200.so")
LIB_CHECKED = os.path.join(HERE, "libdare_b200_checked.so")  # -DDARE_CHECKED: device bounds asserts
SOURCES = ["runtime.cu", "reconstruct.cu", "volume_api.cu", "reslice.cu", "scalar.cu", "merge.cu", "bins.cu",
           "plan.cu", "cells.cu", "similarity.cu", "split.cu"]
HEADERS = ["common.cuh", "volume.cuh", "cells.cuh", "dare_exp.h", "exp_table.h"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "dare_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """libdare_b200.so (or, with checked=True, libdare_b200_checked.so: the same
    sources with -DDARE_CHECKED device-side bounds asserts, for test runs)."""
    lib = LIB_CHECKED if checked else LIB
    if not force and not _stale(lib):
        return lib
    nvcc = nvcc_path()
    objs = []
    build_dir = os.path.join(HERE, "_build_checked" if checked else "_build")
    os.makedirs(build_dir, exist_ok=True)
    common = [
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-std=c++17", "-lineinfo", "-fmad=false",
        "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
        "--expt-relaxed-constexpr",
        "-I", os.path.join(HERE, "..", "include"),
    ]
    if verbose:
        common += ["-Xptxas", "-v"]
    if checked:
        common += ["-DDARE_CHECKED"]
    procs = []
    for src in SOURCES:
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [nvcc, *common, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for cmd, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode != 0:
            sys.stderr.write(out.decode(errors="replace"))
        if p.returncode != 0:
            failed = True
            sys.stderr.write("FAILED: " + " ".join(cmd) + "\n")
    if failed:
        raise RuntimeError("nvcc compilation failed")
    tmp = lib + ".tmp"
    link = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp,
            "-lcudart"]
    subprocess.run(link, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
