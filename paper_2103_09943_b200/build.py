"""Build the sm_100a CUDA library (libfbmp_gpu.so) and the C++ reference-API shim in-tree.

nvcc cross-compiles for sm_100a without a GPU; the .so files are written next to the
sources (paper_2103_09943_b200/lib/) so they travel with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
HOST = os.path.join(HERE, "host")
LIBDIR = os.path.join(HERE, "lib")
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_LIB = "/usr/local/cuda/lib64"
# NCCL: the copy torch ships (same library in the process when torch.distributed is used)
NCCL_DIR = os.path.join(os.path.dirname(os.path.dirname(os.__file__)), "site-packages", "nvidia", "nccl")
if not os.path.isdir(NCCL_DIR):
    import sysconfig
    NCCL_DIR = os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                  "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "--expt-relaxed-constexpr",
                  "-I" + os.path.join(NCCL_DIR, "include")]
CU_SOURCES = ["pansharpen.cu", "kernel_fit.cu", "metrics.cu", "capi.cu"]
GPU_LIB = os.path.join(LIBDIR, "libfbmp_gpu.so")
LINK = ["-L" + CUDA_LIB, "-lcufft", "-lcudart", "-Xlinker", "-rpath," + CUDA_LIB,
        "-L" + os.path.join(NCCL_DIR, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(NCCL_DIR, "lib")]
SHIM_LIB = os.path.join(LIBDIR, "libfbmp.so")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} ... {cmd[-1]}")


def build_gpu(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    headers.append(os.path.join(ROOT, "include", "fbmp_gpu.h"))
    objs, jobs = [], []
    for src in CU_SOURCES:
        sp = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [sp] + headers):
            extra = ["-Xptxas", "-v"] if verbose else []
            jobs.append([NVCC] + NVFLAGS + extra + ["-c", sp, "-o", obj])
    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(_run, jobs))
    if force or jobs or _stale(GPU_LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", GPU_LIB] + objs + LINK)
    return GPU_LIB


SHIM_TEST = os.path.join(LIBDIR, "fbmp_shim_selftest")
CLI = os.path.join(LIBDIR, "fbmp")  # command-line front end (host/fbmp_cli.cpp)


def build_shim(force: bool = False) -> str:
    """libfbmp.so: the reference's fbmp:: C++ API on top of libfbmp_gpu.so (+ its self-test)."""
    srcs = [os.path.join(HOST, "fbmp_api.cpp"), os.path.join(HOST, "raster_io.cpp")]
    hdrs = [os.path.join(ROOT, "include", "fbmp", f) for f in os.listdir(os.path.join(ROOT, "include", "fbmp"))]
    if force or _stale(SHIM_LIB, srcs + hdrs + [GPU_LIB]):
        _run(["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-Wall", "-Wextra",
              "-I" + os.path.join(ROOT, "include"), "-o", SHIM_LIB] + srcs +
             ["-L" + LIBDIR, "-lfbmp_gpu", "-Wl,-rpath,$ORIGIN"])
    test_src = os.path.join(HOST, "shim_selftest.cpp")
    if force or _stale(SHIM_TEST, [test_src, SHIM_LIB] + hdrs):
        _run(["g++", "-O2", "-std=c++20", "-Wall", "-I" + os.path.join(ROOT, "include"), "-o", SHIM_TEST, test_src,
              "-L" + LIBDIR, "-lfbmp", "-lfbmp_gpu", "-Wl,-rpath,$ORIGIN"])
    cli_src = os.path.join(HOST, "fbmp_cli.cpp")
    if os.path.exists(cli_src) and (force or _stale(CLI, [cli_src, SHIM_LIB] + hdrs)):
        _run(["g++", "-O2", "-std=c++20", "-Wall", "-I" + os.path.join(ROOT, "include"), "-o", CLI, cli_src,
              "-L" + LIBDIR, "-lfbmp", "-lfbmp_gpu", "-Wl,-rpath,$ORIGIN"])
    return SHIM_LIB


def build(force: bool = False, verbose: bool = False) -> None:
    build_gpu(force, verbose)
    if os.path.isdir(HOST) and any(f.endswith(".cpp") for f in os.listdir(HOST)):
        build_shim(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(GPU_LIB)
