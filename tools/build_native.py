#!/usr/bin/env python3
"""Build the native library paper_2009_14783_b200/libhetpar_b200.so (sm_100a).

nvcc cross-compiles without a GPU; the CUDA runtime is linked statically so
the library loads on a CPU-only host (every device call then reports
HP_ECUDA), and NCCL is the torch-bundled libnccl.so.2 found through rpath.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2009_14783_b200")
SRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libhetpar_b200.so")
OBJ = os.path.join(ROOT, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        return list(spec.submodule_search_locations)[0]
    raise RuntimeError("NCCL (nvidia.nccl) not found")


def build(verbose: bool = False) -> str:
    # HP_GEMM_PROFILE=1: compile the GEMM's timeline trace / debug hooks in
    # (tools/gemm_trace.py); separate object dir so builds never mix
    profile = os.environ.get("HP_GEMM_PROFILE") == "1"
    # HP_VARIANT=name HP_VARIANT_DEFS="A B": an A/B build with -DA -DB into
    # libhetpar_b200_<name>.so (loaded when HP_LIB_VARIANT=name)
    variant = os.environ.get("HP_VARIANT", "")
    vdefs = ["-D" + d for d in os.environ.get("HP_VARIANT_DEFS", "").split()]
    obj_dir = OBJ + ("_profile" if profile else "") + ("_" + variant if variant else "")
    out = OUT[:-3] + "_" + variant + ".so" if variant else OUT
    os.makedirs(obj_dir, exist_ok=True)
    nd = nccl_dir()
    inc = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include")]
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                    "--expt-relaxed-constexpr"] + inc + (["-DHP_GEMM_PROFILE"] if profile else []) + vdefs
    srcs = sorted(glob.glob(os.path.join(SRC, "*.cu")) + glob.glob(os.path.join(SRC, "*.cpp")))
    hdrs = (glob.glob(os.path.join(SRC, "*.h")) + glob.glob(os.path.join(SRC, "*.cuh")) +
            glob.glob(os.path.join(ROOT, "include", "*.h")))
    newest_hdr = max(os.path.getmtime(h) for h in hdrs)

    def compile_one(src: str) -> str:
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), newest_hdr):
            return obj
        cmd = [NVCC] + flags + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(compile_one, srcs))
    if not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", out] + objs + [
            "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath," + os.path.join(nd, "lib")]
        if verbose:
            print(" ".join(cmd))
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
