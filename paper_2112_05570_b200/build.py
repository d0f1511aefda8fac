"""Build libmwt.so (sm_100a) in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false:
FMA contraction is OFF for every translation unit because the reference
evaluates each fp64 + - * / separately (CPython floats).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_build")
LIB = os.path.join(OUT_DIR, "libmwt.so")
SOURCES = ["mwt_walk.cu", "mwt_struct.cu", "mwt_capi.cu", "mwt_pack.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def flags() -> list[str]:
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "--prec-div=true",
                   "--prec-sqrt=true", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
                   "-ccbin", "/usr/bin/g++", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + ["mwt_internal.h", "mwt_device.cuh"]]
    deps += [os.path.join(ROOT, "include", "mwt.h"), __file__]
    return all(os.path.getmtime(d) <= t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(OUT_DIR, src + ".o")
        cmd = [nvcc()] + flags() + ["-Xptxas", "-v", "-c", os.path.join(CSRC, src), "-o", obj] \
            if src.endswith(".cu") else [nvcc()] + flags() + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        with open(os.path.join(OUT_DIR, src + ".ptxas.txt"), "w") as fh:
            fh.write(r.stderr)
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [nvcc()] + ARCH + ["-shared", "-ccbin", "/usr/bin/g++", "-o", tmp] + objs + ["-lcudart_static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
