"""Build libqlm.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

Each source compiles to its own object in parallel (build/lib_objs/), then one
link; the objects are rebuilt whenever any source or header is newer."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libqlm.so")
OBJ_DIR = os.path.join(ROOT, "build", "lib_objs")
SOURCES = [os.path.join(PKG, "csrc", n) for n in ("qlm_api.cu", "qlm_kernels.cu", "qlm_ws.cu", "qlm_ws2.cu", "qlm_wide.cu", "qlm_req.cu", "qlm_tier.cu", "qlm_group.cu", "qlm_big.cu", "qlm_comm.cu", "qlm_large.cu")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden"]
LDFLAGS = ARCH + ["-shared", "-ldl"]
NVCC_FLAGS = CFLAGS + ["-shared", "-ldl"]   # single-command form (kept for tools)


def _deps():
    return SOURCES + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + \
        glob.glob(os.path.join(PKG, "csrc", "*.h")) + [os.path.join(ROOT, "include", "qlm.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(nvcc):
        nvcc = "nvcc"
    os.makedirs(OBJ_DIR, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include")]
    procs, objs = [], []
    for s in SOURCES:
        o = os.path.join(OBJ_DIR, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        cmd = [nvcc, *CFLAGS, *inc, *(["-Xptxas=-v"] if verbose else []), "-c", "-o", o + ".tmp", s]
        if verbose:
            print(" ".join(cmd))
        procs.append((subprocess.Popen(cmd), o))
    failed = False
    for p, o in procs:
        if p.wait() != 0:
            failed = True
        else:
            os.replace(o + ".tmp", o)
    if failed:
        raise subprocess.CalledProcessError(1, "nvcc (see the compiler output above)")
    tmp = LIB + ".tmp"
    subprocess.check_call([nvcc, *LDFLAGS, "-o", tmp, *objs])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
