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

SOURCES = ["capi.cu", "runtime.cu", "elementwise.cu", "block.cu",
           "block_cluster.cu", "block_chunks.cu", "gemm.cu", "composed.cu", "optim.cu",
           "group.cu", "io.cu"]
HEADERS = ["quant_math.cuh", "kernels.cuh", "runtime.h", "block_common.cuh"]

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


REF = "/root/reference/proj"
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
DROPIN = os.path.join(ROOT, "build", "dropin")


def build_dropin(force=False, verbose=False):
    """TEST ONLY: the reference library with proj/src/quant_ops.cpp replaced
    by the B200 drop-in (csrc/dropin/quant_ops_b200.cpp over liblpq.so), and
    the reference's own unit suites (compiled unchanged against a minimal
    doctest header) and acceptance binary linked against it.  Needs the
    reference sources, so it is built here and the binaries travel."""
    if not os.path.isdir(REF):
        return None
    os.makedirs(DROPIN, exist_ok=True)
    cxx = shutil.which("g++") or "g++"
    inc = ["-I", os.path.join(REF, "include"), "-I", os.path.join(ROOT, "include"),
           "-I", JSON_INC]
    flags = ["-std=c++20", "-O2", "-fPIC", "-w"]
    shim = os.path.join(CSRC, "dropin", "quant_ops_b200.cpp")
    srcs = [os.path.join(REF, "src", f) for f in
            ("tensor.cpp", "enumerate.cpp", "train.cpp", "bench.cpp", "io.cpp")] + [shim]
    objs, jobs = [], []
    for src in srcs:
        o = os.path.join(DROPIN, os.path.basename(src).replace(".cpp", ".o"))
        objs.append(o)
        if force or _newer(o, [src, os.path.join(ROOT, "include", "lpq.h")]):
            jobs.append([cxx, *flags, *inc, "-c", src, "-o", o])
    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    link = ["-L", LIBDIR, "-llpq", f"-Wl,-rpath,{LIBDIR}",
            "-Wl,-rpath,$ORIGIN/../../paper_1910_04540_b200/lib", "-lpthread"]
    main = os.path.join(ROOT, "tests", "native", "doctest_main.cpp")
    tests = [os.path.join(REF, "tests", f) for f in
             ("test_quant_ops.cpp", "test_train.cpp", "test_bench.cpp")]
    tinc = ["-I", os.path.join(ROOT, "tests", "native", "doctest_mini"),
            "-I", os.path.join(REF, "tests")]
    out_t = os.path.join(DROPIN, "lpsim_tests_b200")
    if force or jobs or _newer(out_t, [main, LIB] + tests + objs):
        _run([cxx, *flags, *inc, *tinc, main, *tests, *objs, "-o", out_t, *link], verbose)
    out_a = os.path.join(DROPIN, "lpsim_acceptance_b200")
    acc = os.path.join(REF, "tests", "acceptance.cpp")
    if force or jobs or _newer(out_a, [acc, LIB] + objs):
        _run([cxx, *flags, *inc, *tinc, acc, *objs, "-o", out_a, *link], verbose)
    return out_t, out_a


def build_oracle(verbose=False):
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], verbose)


def build_all(force=False, verbose=False):
    build_oracle(verbose)
    build_host_math(force, verbose)
    lib = build_lib(force, verbose)
    build_dropin(force, verbose)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build_all(a.force, a.verbose))
