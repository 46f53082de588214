"""Builds libsof_cuda.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

The library is the whole product: CUDA kernels + the extern "C" boundary declared
in include/sof_cuda.h. Compiled with --fmad=false so every FP64 expression keeps
the reference's rounding sequence (see csrc/sof_device.cuh).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libsof_cuda.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# tuning experiments: SOF_VARIANT="name:-DKNOB=v ..." builds build/obj_name and
# libsof_cuda_name.so (loaded with SOF_LIB_PATH); the default build is untouched
_VARIANT = os.environ.get("SOF_VARIANT", "")
DEFS: list = []
if _VARIANT:
    _name, _, _defs = _VARIANT.partition(":")
    OBJ = os.path.join(ROOT, "build", "obj_" + _name)
    LIB = os.path.join(PKG, f"libsof_cuda_{_name}.so")
    DEFS = _defs.split()

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
                  "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math", "-Xptxas", "-v"]
# per-file FMA policy: the FP64 parity kernels must not contract
FMAD = {"default": ["--fmad=false"]}


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(ROOT, "include", "sof_cuda.h"))
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src):
    s = os.path.join(CSRC, src)
    o = os.path.join(OBJ, src.replace(".cu", ".o"))
    log = os.path.join(OBJ, src.replace(".cu", ".ptxas.txt"))
    if not _stale(o, [s] + _headers()):
        return o
    cmd = [NVCC] + NVFLAGS + DEFS + FMAD.get(src, FMAD["default"]) + ["-c", s, "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    return o


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(_compile, srcs))
    if _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    if verbose:
        print(f"built {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
