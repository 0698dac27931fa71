"""Build libwsb200.so (the CUDA kernels + C ABI) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_PATH = os.path.join(PKG_DIR, "libwsb200.so")
# translation units and their extra flags: the packed int16 short-read kernels are built with ptxas -O1 (see wsb200_s16.cu)
SOURCES = {"wsb200.cu": [], "wsb200_s16.cu": ["-Xptxas", "-O1"], "hostpack.cpp": []}
DEPS = ["wsb200.cu", "wsb200_s16.cu", "hostpack.cpp", "hostpack.h", "score_kernels.cuh", "score_short.cuh", "score_short16.cuh", "score_short16g.cuh",
        "score_long.cuh", "score_long16.cuh", "traceback_kernels.cuh", "traceback_fill16.cuh", "traceback_host.inl",
        "traceback_band.cuh", "traceback_band_host.inl", os.path.join("..", "..", "include", "wsb200.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def needs_build() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    built = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(os.path.join(CSRC, d)) > built for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    out = out or LIB_PATH
    if force or needs_build() or out != LIB_PATH:
        nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
        extra = os.environ.get("WSB_NVCC_EXTRA", "").split()   # tuning aid, e.g. -DWSB_TG_ONLY
        objdir = os.path.join(PKG_DIR, "csrc", "_obj" + ("" if out == LIB_PATH else "_" + os.path.basename(out)))
        os.makedirs(objdir, exist_ok=True)

        def compile_one(item):
            src, flags = item
            obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
            cmd = [nvcc, *extra, *NVCC_FLAGS, *flags, *(["-Xptxas=-v"] if verbose else []), "-c", "-o", obj, os.path.join(CSRC, src)]
            subprocess.check_call(cmd, cwd=CSRC)
            return obj

        with ThreadPoolExecutor(len(SOURCES)) as pool:
            objs = list(pool.map(compile_one, SOURCES.items()))
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs], cwd=CSRC)
    return out


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose="-v" in sys.argv, out=sys.argv[sys.argv.index("-o") + 1] if "-o" in sys.argv else None))
