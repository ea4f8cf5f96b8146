"""Build libft.so (sm_100a) in-tree with nvcc.

The shared library is the product: the C-ABI of include/ft.h.  It links the
CUDA runtime statically and NCCL (the torch-bundled libnccl.so.2) dynamically.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libft.so")
TORCH_ALLOC_LIB = os.path.join(HERE, "libft_torch_alloc.so")
SOURCES = ["ft_step.cu", "ft_api.cu", "ft_costgen.cu"]
HEADERS = ["ft_kernels.cuh", "ft_step.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl as n  # torch-bundled NCCL (same SONAME torch loads)
        base = list(n.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "ft.h")]
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(d) for d in deps):
        return LIB
    inc, lib = _nccl_dirs()
    cmd = [nvcc(), "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared",
           "-cudart", "static", f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}", "-o", LIB, *srcs,
           f"-L{lib}", "-l:libnccl.so.2", f"-Xlinker", f"-rpath={lib}"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    build_torch_alloc(force=True)
    return LIB


def build_torch_alloc(force: bool = False) -> str:
    """libft_torch_alloc.so: ft_options.alloc/.free backed by torch's CUDA
    caching allocator (csrc/ft_torch_alloc.cpp; links libc10_cuda)."""
    src = os.path.join(CSRC, "ft_torch_alloc.cpp")
    if not force and os.path.exists(TORCH_ALLOC_LIB) and os.path.getmtime(TORCH_ALLOC_LIB) >= os.path.getmtime(src):
        return TORCH_ALLOC_LIB
    import torch
    tdir = os.path.dirname(torch.__file__)
    cuda_inc = os.path.join(os.path.dirname(os.path.dirname(nvcc())) if nvcc() != "nvcc" else "/usr/local/cuda",
                            "include")
    cmd = ["g++", "-std=c++17", "-O2", "-shared", "-fPIC", f"-I{os.path.join(tdir, 'include')}",
           f"-I{cuda_inc}", "-o", TORCH_ALLOC_LIB, src, f"-L{os.path.join(tdir, 'lib')}", "-lc10_cuda",
           "-lc10", f"-Wl,-rpath,{os.path.join(tdir, 'lib')}"]
    subprocess.check_call(cmd)
    return TORCH_ALLOC_LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
