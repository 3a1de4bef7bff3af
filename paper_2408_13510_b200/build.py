"""In-tree build of the engine library `_lib/librs_b200.so` (sm_100a).

    python -m paper_2408_13510_b200.build [-v]

nvcc cross-compiles here without a GPU; the built .so travels to the GPU box
with the repo snapshot.  -fmad=false (and -ffp-contract=off on the host
side) keeps every fp64 multiply and add separately rounded, as the
reference's arithmetic requires.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_lib"
BUILD = PKG / "_build"
INCLUDE = PKG.parent / "include"
LIB = OUT / "librs_b200.so"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "--prec-div=true",
                     "--prec-sqrt=true", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
                     "-Xptxas", "-O3", "-DNDEBUG"]
CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-DNDEBUG"]

CU_SOURCES = ["engine.cu", "host_api.cu"]
CXX_SOURCES = ["workload.cpp"]
HEADERS = ["common.cuh", "predictor.cuh", "replay.cuh", "router.cuh", "mlp.cuh"]


def _digest() -> str:
    h = hashlib.sha256()
    for name in CU_SOURCES + CXX_SOURCES + HEADERS:
        h.update((CSRC / name).read_bytes())
    h.update((INCLUDE / "rs_abi.h").read_bytes())
    h.update(" ".join(NVCC_FLAGS + CXX_FLAGS).encode())
    return h.hexdigest()


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)


def build(verbose: bool = False, force: bool = False, ptxas_verbose: bool = False) -> Path:
    stamp = OUT / ".stamp"
    dig = _digest()
    if not force and LIB.exists() and stamp.exists() and stamp.read_text() == dig:
        return LIB
    BUILD.mkdir(exist_ok=True)
    OUT.mkdir(exist_ok=True)
    objs = []
    extra = ["-Xptxas", "-v"] if ptxas_verbose else []
    for src in CU_SOURCES:
        obj = BUILD / (Path(src).stem + ".o")
        _run([NVCC, *NVCC_FLAGS, *extra, f"-I{INCLUDE}", "-c", str(CSRC / src), "-o", str(obj)],
             verbose or ptxas_verbose)
        objs.append(str(obj))
    for src in CXX_SOURCES:
        obj = BUILD / (Path(src).stem + ".o")
        _run([CXX, *CXX_FLAGS, f"-I{INCLUDE}", "-c", str(CSRC / src), "-o", str(obj)], verbose)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs, "-lpthread"],
         verbose)
    tmp.replace(LIB)
    stamp.write_text(dig)
    return LIB


if __name__ == "__main__":
    v = "-v" in sys.argv
    print(build(verbose=v, force="-f" in sys.argv, ptxas_verbose="--ptxas" in sys.argv))
