"""Build libasim.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

Every source compiles to its own object in parallel (build/), then one nvcc
link produces the shared library with the CUDA runtime linked statically."""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libasim.so")
SOURCES = ["ctx.cpp", "search.cpp", "chunked.cpp", "sim.cu", "chunk.cu", "batch.cu"]
HEADERS = ["asim_internal.h", "ctx.h", "launch_cache.h", "chunk_common.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-Wall",
          "--expt-relaxed-constexpr"]
LDFLAGS = ["-shared", "-cudart", "static"]


def _inputs():
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "asim.h"))
    files.append(os.path.abspath(__file__))
    return files


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build(force: bool = False, verbose: bool = False, extra=()) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    tag = f"{os.getpid()}"

    def compile_one(src):
        obj = os.path.join(OBJ, f"{os.path.splitext(src)[0]}.{tag}.o")
        # .cpp sources are host code that calls the CUDA runtime: nvcc -x cu
        # would also work, but plain host compilation keeps them out of cicc
        cmd = [NVCC, *ARCH, *CFLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c",
               "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        return obj

    # the heaviest translation units first
    order = sorted(SOURCES, key=lambda f: -os.path.getsize(os.path.join(CSRC, f)))
    with ThreadPoolExecutor(max_workers=min(len(order), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, order))
    tmp = LIB + f".tmp{tag}"
    cmd = [NVCC, *ARCH, *LDFLAGS, "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    for o in objs:
        os.remove(o)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          extra=["-Xptxas", "-v"] if "--ptxas-v" in sys.argv else [])
    print(LIB)
