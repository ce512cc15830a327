"""Build libss_b200.so in-tree with nvcc for sm_100a (no JIT, no torch
extension machinery): one object per .cu, linked into a C-ABI shared
library that the host mirror loads with ctypes."""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libss_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["abi.cu", "preprocess.cu", "binning.cu", "raster_fwd.cu", "raster_bwd.cu", "chain_bwd.cu",
           "env.cu", "optim.cu", "train_step.cu", "losses.cu", "knn.cu", "refine.cu", "grid.cu"]
# preprocess mirrors numpy float32 expression by expression: no contraction
NO_FMAD = {"preprocess.cu"}

BASE_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-ccbin", "/usr/bin/g++", "-I", os.path.join(HERE, "..", "include")]


def _compile(src, verbose=False):
    obj = os.path.join(OUT_DIR, src.replace(".cu", ".o"))
    flags = list(BASE_FLAGS) + os.environ.get("SS_NVCC_FLAGS", "").split()  # experiment switches (-D...)
    if src in NO_FMAD:
        flags.append("-fmad=false")
    if verbose:
        flags += ["-Xptxas", "-v"]
    cmd = [NVCC, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


STAMP = LIB + ".flags"


def _flag_key():
    """What the .so was built with: the base flags plus the experiment
    switches (SS_NVCC_FLAGS).  Stored next to the library; a differing key
    forces a rebuild, so a variant build (e.g. -DSS_UNIFORM_BOUNDS from a
    tools/ script) is never shipped by a later default build()."""
    return " ".join(BASE_FLAGS + os.environ.get("SS_NVCC_FLAGS", "").split())


def _stale():
    if not os.path.exists(LIB):
        return True
    try:
        with open(STAMP) as f:
            if f.read() != _flag_key():
                return True
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "ss_abi.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    if verbose:
        for _, err in results:
            sys.stderr.write(err)
    objs = [o for o, _ in results]
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-ccbin", "/usr/bin/g++",
           "-o", LIB, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    with open(STAMP, "w") as f:
        f.write(_flag_key())
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
