"""Build librte_b200.so (CUDA kernels for sm_100a + C-ABI) in-tree with nvcc.

Usage: python -m paper_2402_10488_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# Development variants: RTE_BUILD_DEFINES="-DNAME ..." builds into
# RTE_BUILD_OUT (a separate library path, with its own object directory).
DEFINES = os.environ.get("RTE_BUILD_DEFINES", "").split()
LIB = os.environ.get("RTE_BUILD_OUT") or os.path.join(HERE, "librte_b200.so")
BUILD = os.path.join(HERE, "_build") if not os.environ.get("RTE_BUILD_OUT") else LIB + ".objs"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]
SOURCES = ["capi.cu", "sweep1d.cu", "si1d.cu", "sweep2d.cu", "dsa1d.cu", "dsa2d.cu", "rom.cu", "kinetic.cu", "pod.cu", "gmres.cu", "setup.cpp"]


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, force):
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
    deps = [path, os.path.join(os.path.dirname(HERE), "include", "rte_b200.h")] + \
        [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    if not force and not _stale(obj, deps):
        return obj, ""
    # host setup helpers: OpenMP; no FMA contraction (bitwise the numpy / reference arithmetic)
    omp = ["-Xcompiler", "-fopenmp", "-Xcompiler", "-ffp-contract=off"] if src.endswith(".cpp") else []
    cmd = [NVCC] + ARCH + FLAGS + DEFINES + omp + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s%s" % (src, r.stdout, r.stderr))
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force), SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for o, log in results:
            if log:
                print("==", os.path.basename(o), "\n", log)
    if force or _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-lgomp", "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n%s%s" % (r.stdout, r.stderr))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
