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
STATS_LIB_PATH = PKG / "libzd_stats.so"   # profiling variant (-DZD_KNN_STATS work counters)
SOURCES = ["sort.cu", "tree.cu", "knn.cu", "knn_warp.cu", "update.cu", "incr.cu", "api.cu"]
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


def stale(path: Path = LIB_PATH) -> bool:
    if not path.exists():
        return True
    t = path.stat().st_mtime
    deps = [CSRC / f for f in DEPS] + [ROOT / "include" / "zd.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build_lib(force: bool = False, verbose: bool = False, stats: bool = False, defines=(), out=None) -> Path:
    """Build libzd.so (or, for experiments, a variant with extra -D defines at `out`)."""
    path = Path(out).resolve() if out else (STATS_LIB_PATH if stats else LIB_PATH)
    if not force and not stale(path):
        return path
    tmp = path.with_name(f"{path.name}.tmp{os.getpid()}")
    cmd = [_nvcc(), *NVCC_FLAGS, *(["-DZD_KNN_STATS"] if stats else []), *[f"-D{d}" for d in defines],
           *[str(CSRC / s) for s in SOURCES], "-o", str(tmp)]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd, cwd=str(CSRC))
    os.replace(tmp, path)
    return path
