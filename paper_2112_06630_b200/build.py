"""Build libknng_cuda.so in-tree with nvcc for sm_100a (no JIT cache, no torch).

    python -m paper_2112_06630_b200.build [--verbose]

Objects go to paper_2112_06630_b200/build/, the shared library to
paper_2112_06630_b200/lib/libknng_cuda.so (git-ignored; travels to the GPU
box with the gpurun snapshot).  Rebuilds only what changed.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "lib", "libknng_cuda.so")
DIAG = os.path.join(PKG, "lib", "libknng_diag.so")  # FFMA peak probe (bench only)
CLI = os.path.join(ROOT, "proj", "tools", "build", "knng_cuda_cli")  # build / recall front end
SOURCES = ["graph_kernels.cu", "join.cu", "join5.cu", "join_gl.cu", "join_tc.cu", "join_u8.cu", "join_u8_tc.cu", "bruteforce.cu", "reorder.cu", "host_io.cu", "api.cu"]
HEADERS = ["common.cuh", "kernels.cuh", "tile_math.cuh", "join5_geom.cuh"]
# join.cu: no FMA contraction anywhere, so the unfused (multiply, then add)
# distance path stays unfused at the SASS level; explicit fma intrinsics are
# unaffected (SURVEY.md §8a-6 bit-exactness)
PER_FILE = {"join.cu": ["--fmad=false"], "join5.cu": ["--fmad=false"], "join_gl.cu": ["--fmad=false"], "join_tc.cu": ["--fmad=false"]}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "knng_cuda.h")]
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = [nvcc(), *ARCH, *FLAGS, *PER_FILE.get(src, []), "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    # the CLI front end (proj/tools), against the C-ABI only
    cli_src = os.path.join(ROOT, "proj", "tools", "knng_cuda_cli.cpp")
    if force or _stale(CLI, [cli_src, LIB, os.path.join(ROOT, "include", "knng_cuda.h")]):
        os.makedirs(os.path.dirname(CLI), exist_ok=True)
        cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-o", CLI, cli_src,
               "-L", os.path.dirname(LIB), "-lknng_cuda",
               "-Wl,-rpath," + os.path.relpath(os.path.dirname(LIB), os.path.dirname(CLI)).join(
                   ["$ORIGIN/", ""])]
        subprocess.run(cmd, check=True)
    diag_src = os.path.join(CSRC, "diag.cu")
    if force or _stale(DIAG, [diag_src]):
        cmd = [nvcc(), *ARCH, *FLAGS, "-shared", "-o", DIAG, diag_src, "-cudart", "static"]
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build(verbose=a.verbose, force=a.force))
    sys.exit(0)
