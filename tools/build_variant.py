"""Build an A/B variant of libekya.so with extra nvcc flags (tools only; the product loads
paper_2012_10557_b200/libekya.so).  usage: [EKYA_VARIANT_CSRC=DIR] python tools/build_variant.py OUT.so -DFLAG=..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2012_10557_b200 import build as B  # noqa: E402

out, extra = sys.argv[1], sys.argv[2:]
inc, lib = B._nccl_dirs()
objdir = os.path.join("/tmp", "ekya_variant_" + os.path.basename(out))
os.makedirs(objdir, exist_ok=True)
common = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
          "-Xcompiler", "-fPIC", "-I", inc, "-I", os.path.join(B.ROOT, "include"), *extra]
objs = []
for src in B.SOURCES:
    obj = os.path.join(objdir, src.replace(".cu", ".o"))
    csrc = os.environ.get("EKYA_VARIANT_CSRC", B.CSRC)   # another source tree (A/B of a code change)
    subprocess.run(["nvcc", *common, "-I", B.CSRC, "-c", os.path.join(csrc, src), "-o", obj], check=True)
    objs.append(obj)
rt = B._nvidia_lib("cuda_runtime")
subprocess.run(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out, *objs, "-L", lib,
                "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib] + (["-Xlinker", "-rpath=" + rt] if rt else []) +
               ["-cudart", "shared"], check=True)
print(out)
