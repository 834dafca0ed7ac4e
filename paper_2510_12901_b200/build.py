"""Build libsimuli.so in-tree: nvcc for sm_100a (tcgen05-era Blackwell) + g++ host code.

Kernels are compiled with ``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo``;
host code that produces interface-defined float32 values (tiling, depth-key origin) is
built with ``-ffp-contract=off`` so no FMA contraction changes a bit.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsimuli.so")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")

CU_SOURCES = ["project.cu", "binsort.cu", "render.cu", "backward.cu"]
CPP_SOURCES = ["tiling_host.cpp", "abi.cpp"]
HEADERS = ["common.cuh", "camera.cuh", "abi_util.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# approximate float division / square root and flushed denormals (the interface-defined
# values -- depth keys, tile maps, box-edge shifts -- use explicit __f*_rn intrinsics and are
# unaffected by -prec-*; measured on config B: projection 206 -> 194 us, LiDAR render 202 ->
# 182 us).  The backward replays the render's float32 response arithmetic, so it is built
# with the same flags.
_FAST = ["-ftz=true", "-prec-div=false", "-prec-sqrt=false"]
FAST_FLAGS = {"project.cu": _FAST, "render.cu": _FAST, "backward.cu": _FAST}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src, os.path.abspath(__file__)] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "simuli.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, src + ".o")
    if not _stale(obj, path):
        return obj
    if src.endswith(".cu"):
        cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
               "-Xptxas", "-v" if verbose else "-O3", "-I", INCLUDE, *FAST_FLAGS.get(src, []), "-c", path, "-o", obj]
        # profiling builds only (e.g. SIMULI_EXTRA_NVCC=-DSIMULI_RENDER_PROFILE, with build(force=True))
        cmd += os.environ.get("SIMULI_EXTRA_NVCC", "").split()
    else:
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall",
               "-I", INCLUDE, "-I", "/usr/local/cuda/include", "-c", path, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    if force:
        for f in os.listdir(BUILD):
            os.remove(os.path.join(BUILD, f))
    with cf.ThreadPoolExecutor(max_workers=len(CU_SOURCES) + len(CPP_SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), CU_SOURCES + CPP_SOURCES))
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread", "-ldl", "-lrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
