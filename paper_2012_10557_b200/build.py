"""Build libekya.so (sm_100a) in-tree with nvcc.

Flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo, -fmad=false
(no FMA contraction anywhere: DESIGN.md section 2), no fast-math.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libekya.so")
SOURCES = ["api.cu", "eval.cu", "thief.cu", "profile.cu", "comm.cu", "place.cu", "baselines.cu", "window.cu"]
HEADERS = ["ekya_common.cuh", "stream_tables.cuh", "launch.h"]


def _nvidia_lib(name):
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, name, "lib")
        if os.path.isdir(d):
            return d
    return None


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for base in spec.submodule_search_locations:
            cands.append(os.path.join(base, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("nccl.h not found (expected the torch-bundled nvidia/nccl package)")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "ekya.h"),
                                                                  __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    inc, lib = _nccl_dirs()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
              "-std=c++17", "-Xcompiler", "-fPIC", "-I", inc, "-I", os.path.join(ROOT, "include")]
    if verbose:
        common += ["-Xptxas", "-v"]
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        subprocess.run([nvcc, *common, "-c", os.path.join(CSRC, src), "-o", obj], check=True)
        objs.append(obj)
    rt = _nvidia_lib("cuda_runtime")   # the libcudart torch itself loads: one runtime per process
    rt_rpath = ["-Xlinker", "-rpath=" + rt] if rt else []
    tmp = LIB + ".tmp"
    subprocess.run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs,
                    "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib, *rt_rpath,
                    "-cudart", "shared"], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
