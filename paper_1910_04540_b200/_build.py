"""Build recipe for liblpq.so (sm_100a) and the test-side native helpers.

    python -m paper_1910_04540_b200._build          # incremental
    python -m paper_1910_04540_b200._build --force

Outputs (all in-tree, git-ignored, shipped to the GPU box with the tree):
    paper_1910_04540_b200/lib/liblpq.so      the product library (include/lpq.h)
    build/libquant_math_host.so              TEST ONLY: the kernels' element
                                             math compiled for the host CPU
    oracle/liblpq_oracle.so, oracle/_ref/... TEST ONLY: CPU checkers
                                             (oracle/Makefile)

Compilation: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo,
--fmad=false (no FMA contraction may change a rounding), no fast-math, IEEE
denormals; cudart linked statically so the library loads beside torch.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(LIBDIR, "liblpq.so")
HOST_MATH = os.path.join(ROOT, "build", "libquant_math_host.so")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")

SOURCES = ["capi.cu", "runtime.cu", "elementwise.cu", "block.cu", "gemm.cu",
           "composed.cu"]
HEADERS = ["quant_math.cuh", "kernels.cuh", "runtime.h"]

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "--fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "-Xptxas", "-warn-spills",
    "-I", os.path.join(ROOT, "include"),
]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)
    return r


def build_lib(force=False, verbose=False):
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "lpq.h")]
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJDIR, src.replace(".cu", ".o"))
        if force or _newer(o, [s] + hdrs):
            jobs.append([NVCC, *NVCC_FLAGS, "-c", s, "-o", o])
    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    objs = [os.path.join(OBJDIR, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or _newer(LIB, objs):
        _run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
              "-o", LIB + ".tmp", *objs, "-lpthread"], verbose)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def build_host_math(force=False, verbose=False):
    src = os.path.join(ROOT, "tests", "native", "host_math_capi.cpp")
    if not os.path.exists(src):
        return None
    os.makedirs(os.path.dirname(HOST_MATH), exist_ok=True)
    if force or _newer(HOST_MATH, [src, os.path.join(CSRC, "quant_math.cuh")]):
        cxx = shutil.which("g++") or "g++"
        _run([cxx, "-std=c++17", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
              "-fno-fast-math", "-frounding-math", "-o", HOST_MATH, src], verbose)
    return HOST_MATH


def build_oracle(verbose=False):
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], verbose)


def build_all(force=False, verbose=False):
    build_oracle(verbose)
    build_host_math(force, verbose)
    return build_lib(force, verbose)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build_all(a.force, a.verbose))
