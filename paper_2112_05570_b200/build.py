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


def build_id(defines: list[str] | None = None) -> str:
    """sha256 of the sources, headers, flags and defines (deterministic, unlike
    the linked binary): mwt_build_id() of the library built from them."""
    import hashlib
    h = hashlib.sha256()
    for f in SOURCES + ["mwt_internal.h", "mwt_device.cuh"]:
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(f.encode() + b"\0" + fh.read())
    with open(os.path.join(ROOT, "include", "mwt.h"), "rb") as fh:
        h.update(fh.read())
    h.update(" ".join(flags() + sorted(defines or [])).replace(ROOT, "").encode())
    return h.hexdigest()[:32]


def build(force: bool = False, verbose: bool = False, out_dir: str | None = None,
          defines: list[str] | None = None) -> str:
    """Build into _build/ (or ``out_dir``: an A/B variant with extra ``-D``
    ``defines``, e.g. ab/<tag>/libmwt.so; never the shipped library)."""
    out_dir = out_dir or OUT_DIR
    lib = os.path.join(out_dir, "libmwt.so")
    if out_dir == OUT_DIR and not defines and not force and up_to_date():
        return LIB
    os.makedirs(out_dir, exist_ok=True)
    extra = ["-D" + d for d in (defines or [])] + [f'-DMWT_BUILD_ID="{build_id(defines)}"']
    objs = []
    for src in SOURCES:
        obj = os.path.join(out_dir, src + ".o")
        cmd = [nvcc()] + flags() + extra + ["-Xptxas", "-v", "-c", os.path.join(CSRC, src), "-o", obj] \
            if src.endswith(".cu") else [nvcc()] + flags() + extra + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        with open(os.path.join(out_dir, src + ".ptxas.txt"), "w") as fh:
            fh.write(r.stderr)
        objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [nvcc()] + ARCH + ["-shared", "-ccbin", "/usr/bin/g++", "-o", tmp] + objs + ["-lcudart_static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python build.py [--force] [-v] [--out DIR -DNAME[=V] ...]
    a = sys.argv[1:]
    out = a[a.index("--out") + 1] if "--out" in a else None
    print(build(force="--force" in a, verbose="-v" in a, out_dir=out,
                defines=[x[2:] for x in a if x.startswith("-D")]))
