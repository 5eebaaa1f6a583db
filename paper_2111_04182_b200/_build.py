"""Builds libzd.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_PATH = PKG / "libzd.so"
SOURCES = ["sort.cu", "tree.cu", "knn.cu", "update.cu", "api.cu"]
DEPS = SOURCES + ["common.cuh", "internal.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xcompiler", "-fvisibility=hidden",   # only the extern "C" zd_* API is exported
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or Path(c).exists()):
            return c
    return "nvcc"


def stale() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    deps = [CSRC / f for f in DEPS] + [ROOT / "include" / "zd.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build_lib(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB_PATH
    tmp = LIB_PATH.with_name(f"libzd.so.tmp{os.getpid()}")
    cmd = [_nvcc(), *NVCC_FLAGS, *[str(CSRC / s) for s in SOURCES], "-o", str(tmp)]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd, cwd=str(CSRC))
    os.replace(tmp, LIB_PATH)
    return LIB_PATH
