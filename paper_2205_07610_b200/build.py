"""Build libwsb200.so (the CUDA kernels + C ABI) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_PATH = os.path.join(PKG_DIR, "libwsb200.so")
SOURCES = ["wsb200.cu"]
DEPS = ["wsb200.cu", "score_kernels.cuh", "score_short.cuh", "score_short16.cuh", "score_short16g.cuh", "score_long.cuh", "score_long16.cuh", "traceback_kernels.cuh", "traceback_fill16.cuh", "traceback_host.inl", "traceback_band.cuh", "traceback_band_host.inl",
        os.path.join("..", "..", "include", "wsb200.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def needs_build() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    built = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(os.path.join(CSRC, d)) > built for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
        cmd = [nvcc, *NVCC_FLAGS, "-o", LIB_PATH, *[os.path.join(CSRC, s) for s in SOURCES]]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        extra = os.environ.get("WSB_NVCC_EXTRA", "").split()   # tuning aid, e.g. -DWSB_TG_ONLY
        cmd[1:1] = extra
        subprocess.check_call(cmd, cwd=CSRC)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force=True, verbose=True))
