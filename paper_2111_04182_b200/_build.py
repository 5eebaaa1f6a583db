"""Builds libzd.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import shutil
import subprocess
import tempfile
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
    """Build libzd.so (or, for experiments, a variant with extra -D defines at `out`).
    Each translation unit is compiled in parallel (nvcc -c), then linked with nvcc."""
    path = Path(out).resolve() if out else (STATS_LIB_PATH if stats else LIB_PATH)
    if not force and not stale(path):
        return path
    tag = f"{path.stem}.{os.getpid()}"
    objdir = Path(tempfile.mkdtemp(prefix=f"zdobj_{tag}_"))
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    extra = [*(["-DZD_KNN_STATS"] if stats else []), *[f"-D{d}" for d in defines]]
    procs = []
    for s in SOURCES:
        cmd = [_nvcc(), *flags, *extra, "-c", str(CSRC / s), "-o", str(objdir / (s + ".o"))]
        if verbose:
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd, cwd=str(CSRC))))
    for cmd, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    tmp = path.with_name(f"{path.name}.tmp{os.getpid()}")
    link = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
            *[str(objdir / (s + ".o")) for s in SOURCES], "-o", str(tmp)]
    if verbose:
        print(" ".join(link))
    subprocess.check_call(link, cwd=str(CSRC))
    os.replace(tmp, path)
    shutil.rmtree(objdir, ignore_errors=True)
    return path
