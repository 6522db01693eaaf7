"""Builds the in-tree CUDA library ``libflowfem_b200.so`` for sm_100a with nvcc.

Kernels that must reproduce the reference's x86-64 (-O2, no FMA) arithmetic bit for bit
(imaging, operator, adapt) are compiled with ``--fmad=false``; the band factor/solve and
the CG kernels keep FMA contraction. Objects are rebuilt when their sources are newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
BUILD = os.path.join(HERE, "_build_prof" if os.environ.get("FFB_PROFILE") else "_build")
LIB = os.environ.get("FFB_LIB_OUT", os.path.join(HERE, "libflowfem_b200.so"))

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-I", CSRC,
          "-I", os.path.join(ROOT, "include")]
if os.environ.get("FFB_PROFILE"):
    COMMON.append("-DFFB_PROFILE")
COMMON += os.environ.get("FFB_NVCC_FLAGS", "").split()  # development experiments (-D...)
CU = {
    "imaging.cu": ["--fmad=false"],
    "operator.cu": ["--fmad=false"],
    "adapt.cu": ["--fmad=false"],
    "band.cu": ["-Xptxas", "-v"] if os.environ.get("FFB_PTXAS_V") else [],
    "pcg.cu": [],
    "coarse.cu": [],
    "comm.cu": [],
    "ras.cu": ["--fmad=false"],
    "linsolve.cu": ["--fmad=false"],
    "metrics.cu": ["--fmad=false"],
}
CPP = ["capi.cpp", "partition.cpp", "rcm.cpp", "io.cpp"]
HEADERS = ["ffb_internal.cuh", "partition.hpp", "comm.hpp"]


def _newer(src_list, dst):
    if not os.path.exists(dst):
        return True
    t = os.path.getmtime(dst)
    return any(os.path.getmtime(s) > t for s in src_list)


def _compile(src, extra):
    obj = os.path.join(BUILD, src + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "flowfem_b200.h")]
    if not _newer(deps, obj):
        return obj, None
    cmd = [NVCC] + ARCH + COMMON + extra + ["-c", os.path.join(CSRC, src), "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, "-x", "cu"] + ARCH + COMMON + ["-c", os.path.join(CSRC, src), "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{p.stdout}\n{p.stderr}")
    return obj, (p.stdout + p.stderr).strip() or None


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    jobs = [(s, e) for s, e in CU.items()] + [(s, []) for s in CPP]
    with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
        res = list(ex.map(lambda j: _compile(*j), jobs))
    objs = [o for o, _ in res]
    for (src, _), (_, log) in zip(jobs, res):
        if verbose and log:
            print(f"[{src}] {log}", file=sys.stderr)
    if _newer(objs, LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt", "-ldl",
                                                             "-lpthread", "-lz"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stdout}\n{p.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
