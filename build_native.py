"""Builds the three native libraries in-tree (they travel to the GPU box).

- paper_1607_06618_b200/_lib/libgerbil.so : the product (C ABI, sm_100a kernels)
- synth/libsynth.so                       : synthetic input generator (host + device twin)
- oracle/liboracle.so                     : the CPU oracle (test infrastructure only)

nvcc cross-compiles for sm_100a without a GPU (`-gencode arch=compute_100a,code=sm_100a`).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1607_06618_b200")
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
OBJDIR = os.path.join(ROOT, "build", "obj")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
           "-I" + os.path.join(ROOT, "include")] + ARCH
# tuning experiments only: extra nvcc flags (e.g. -DGERBIL_SM_MINB=4) force a rebuild
EXTRA = os.environ.get("GERBIL_NVCC_EXTRA", "").split()
NVFLAGS += EXTRA

GERBIL_CU = ["parse.cu", "supermer.cu", "supermer_reads.cu", "ordering.cu", "shuffle.cu", "count.cu", "count_wide.cu", "count_smem.cu", "count_ref.cu", "sort.cu", "compact.cu", "comm.cu", "waves.cu", "pipeline.cu", "io.cu", "spill.cu", "results.cu",
             "api.cu"]
GERBIL_CPP = ["reader.cpp", "output.cpp"]

LIB_GERBIL = os.path.join(LIBDIR, "libgerbil.so")
LIB_SYNTH = os.path.join(ROOT, "synth", "libsynth.so")
LIB_ORACLE = os.path.join(ROOT, "oracle", "liboracle.so")


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} … {cmd[-1]}")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers(d: str) -> list[str]:
    return [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".h", ".cuh"))]


def build_gerbil(force: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    hdrs = _headers(CSRC) + [os.path.join(ROOT, "include", "gerbil.h")]
    srcs = [os.path.join(CSRC, f) for f in GERBIL_CU + GERBIL_CPP]
    force = force or bool(EXTRA)
    if not force and not _stale(LIB_GERBIL, srcs + hdrs):
        return LIB_GERBIL
    jobs = []
    objs = []
    for f in GERBIL_CU:
        o = os.path.join(OBJDIR, f + ".o")
        objs.append(o)
        if force or _stale(o, [os.path.join(CSRC, f)] + hdrs):
            jobs.append([NVCC, *NVFLAGS, "-c", os.path.join(CSRC, f), "-o", o])
    for f in GERBIL_CPP:
        o = os.path.join(OBJDIR, f + ".o")
        objs.append(o)
        if force or _stale(o, [os.path.join(CSRC, f)] + hdrs):
            jobs.append(["g++", "-O3", "-std=c++20", "-fPIC", "-pthread", "-c",
                         os.path.join(CSRC, f), "-o", o])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(_run, jobs))
    _run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", LIB_GERBIL,
          "-ldl", "-lpthread", "-lz"])
    return LIB_GERBIL


def build_synth(force: bool = False) -> str:
    src = os.path.join(ROOT, "synth", "synth.cu")
    deps = [src, os.path.join(ROOT, "synth", "synth_core.h")]
    if force or _stale(LIB_SYNTH, deps):
        _run([NVCC, *NVFLAGS, "-shared", src, "-o", LIB_SYNTH, "-lpthread"])
    return LIB_SYNTH


def build_oracle(force: bool = False) -> str:
    src = os.path.join(ROOT, "oracle", "oracle.cpp")
    if force or _stale(LIB_ORACLE, [src]):
        _run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", src, "-o", LIB_ORACLE])
    return LIB_ORACLE


def build_all(force: bool = False) -> None:
    with cf.ThreadPoolExecutor(max_workers=3) as ex:
        futs = [ex.submit(build_gerbil, force), ex.submit(build_synth, force),
                ex.submit(build_oracle, force)]
        for f in futs:
            f.result()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built:", LIB_GERBIL, LIB_SYNTH, LIB_ORACLE)
