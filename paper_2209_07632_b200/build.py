"""Compile libvf.so in-tree for sm_100a (nvcc -gencode arch=compute_100a,code=sm_100a).

Each source is compiled to an object under build/ (rebuilt when it or a
header is newer), in parallel, then linked.

Usage: python -m paper_2209_07632_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libvf.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", *ARCH, "-lineinfo"]
# host code: AVX2; no FMA contraction where the build must reproduce the
# visibility predicate and F_ij bit for bit (reading R-VIS); the rank
# estimation (vf_svd.cpp) may contract.
HOST = {"vf_svd.cpp": "-fPIC,-fopenmp,-mavx2,-mfma,-ffp-contract=fast"}
HOST_DEFAULT = "-fPIC,-fopenmp,-mavx2,-ffp-contract=off"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cpp")) + glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(HERE, "..", "include", "vf.h")]


def _obj(src):
    return os.path.join(OBJ, os.path.basename(src) + ".o")


def _newer(a, deps):
    if not os.path.exists(a):
        return True
    t = os.path.getmtime(a)
    return any(os.path.getmtime(d) > t for d in deps)


def stale() -> bool:
    return _newer(LIB, sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    hdr = headers() + [__file__]
    todo = [s for s in sources() if force or _newer(_obj(s), [s] + hdr)]

    def compile_one(src):
        cmd = [NVCC, *FLAGS, "-Xcompiler", HOST.get(os.path.basename(src), HOST_DEFAULT), "-c", src, "-o", _obj(src)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)

    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        list(ex.map(compile_one, todo))
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp,
                           *[_obj(s) for s in sources()], "-lgomp", "-ldl", "-lcublas", "-lcusolver", "-lcusparse",
                           "-Xlinker", "-rpath,/usr/local/cuda/lib64"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
