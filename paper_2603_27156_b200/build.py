"""In-tree build of the sm_100a CUDA library (libgsrcuda.so).

nvcc cross-compiles for sm_100a without a GPU. Objects are rebuilt only when
their sources change, so the driver's build() check stays fast.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libgsrcuda.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]
SOURCES = ["kernels.cu", "tile_w32.cu", "tile_w64.cu", "tile_w128.cu", "fast.cu", "capi.cu"]
HEADERS = ["kernels.cuh", "common.cuh", "tile.cuh", os.path.join(ROOT, "include", "gsr_cuda.h")]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build(verbose: bool = False) -> str:
    os.makedirs(os.path.join(CSRC, "_obj"), exist_ok=True)
    hdr_t = max(_mtime(os.path.join(CSRC, h)) if not os.path.isabs(h) else _mtime(h) for h in HEADERS)
    objs, todo = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(CSRC, "_obj", src.replace(".cu", ".o"))
        objs.append(o)
        if _mtime(o) < max(_mtime(s), hdr_t):
            todo.append([NVCC, *ARCH, *FLAGS, "-c", s, "-o", o])
    from concurrent.futures import ThreadPoolExecutor
    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        list(ex.map(run, todo))
    if _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-Xcompiler", "-fPIC", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    build_cli(verbose)
    return LIB


CLI_SRC = os.path.join(ROOT, "tools", "gsrnet_cuda.cpp")
CLI = os.path.join(ROOT, "tools", "gsrnet-cuda")


def build_cli(verbose: bool = False) -> str:
    """C++ host CLI over the C-ABI (include/gsr/cuda_api.hpp), linked to libgsrcuda.so."""
    deps = [CLI_SRC, os.path.join(ROOT, "include", "gsr", "cuda_api.hpp"), os.path.join(ROOT, "include", "gsr", "common.hpp"), LIB]
    if _mtime(CLI) >= max(_mtime(d) for d in deps):
        return CLI
    cmd = ["g++", "-O2", "-std=c++20", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           CLI_SRC, "-o", CLI, "-L", HERE, "-lgsrcuda", "-Wl,-rpath,$ORIGIN/../paper_2603_27156_b200"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    return CLI


if __name__ == "__main__":
    print(build(verbose=True))
