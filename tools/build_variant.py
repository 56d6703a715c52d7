"""Build an experimental variant of libfbmp_gpu.so with extra nvcc -D flags (A/B timing only):
    python tools/build_variant.py NAME -DFOO=1 ...  ->  paper_2103_09943_b200/lib/exp/libfbmp_gpu_NAME.so
Load it with FBMP_GPU_LIB=<path>."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2103_09943_b200"))
import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
bdir = os.path.join(B.BUILD, "variant_" + name)
os.makedirs(bdir, exist_ok=True)
os.makedirs(os.path.join(B.LIBDIR, "exp"), exist_ok=True)
objs = []
for src in B.CU_SOURCES:
    obj = os.path.join(bdir, src.replace(".cu", ".o"))
    subprocess.run([B.NVCC] + B.NVFLAGS + defs + ["-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
    objs.append(obj)
out = os.path.join(B.LIBDIR, "exp", f"libfbmp_gpu_{name}.so")
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", out] + objs + B.LINK, check=True)
print(out)
