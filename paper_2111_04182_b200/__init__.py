"""B200-native zd-tree (Blelloch & Dobson, arXiv 2111.04182) — Python binding.

Thin ctypes binding over the C ABI in include/zd.h (libzd.so, hand-written sm_100a
CUDA).  It only marshals arguments: every step of the hot path runs in the CUDA
kernels.  There is no CPU fallback: if libzd.so is missing or cannot be loaded,
load() raises.

Arrays may be torch tensors (CUDA or CPU) or numpy arrays; CUDA tensors are passed
as device pointers, host arrays as host pointers (the library stages them).
Work runs on torch's current CUDA stream at build time unless a stream is given.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

import os
from pathlib import Path

from ._build import LIB_PATH, STATS_LIB_PATH, build_lib

ZD_OK, ZD_EINVAL, ZD_ERANGE, ZD_ENOMEM, ZD_ECUDA = 0, -1, -2, -3, -4
ZD_K_MAX = 128
ZD_KNN_ROOT_BASED = 1
ZD_KNN_WARP = 2
ZD_LEAF_MAX_MAX = 32
PHASES = ("sort", "topology", "bbox", "merge_compact", "knn", "validate")

_lib = None


class ZdError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Opts(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("leaf_max", C.c_int), ("timing", C.c_int), ("shift_set", C.c_int),
                ("shift", C.c_int32 * 3)]


class _Info(C.Structure):
    _fields_ = [("dim", C.c_int), ("leaf_max", C.c_int), ("n", C.c_int64), ("n_next", C.c_int64),
                ("n_leaves", C.c_int64), ("n_internal", C.c_int64), ("root", C.c_int32),
                ("node_words", C.c_int32), ("shift", C.c_int32 * 3), ("fast_inserts", C.c_int64), ("fast_deletes", C.c_int64),
                ("sort_fallbacks", C.c_int64)]


def load():
    """Load libzd.so (never rebuilt here).  ZD_LIB=stats selects the profiling variant
    libzd_stats.so (work counters, zd_knn_stats); ZD_LIB=<path>.so an experiment build."""
    global _lib
    if _lib is not None:
        return _lib
    sel = os.environ.get("ZD_LIB", "")
    path = STATS_LIB_PATH if sel == "stats" else (Path(sel) if sel.endswith(".so") else LIB_PATH)
    if not path.exists():
        raise RuntimeError(f"{path.name} not built ({path}); run __graft_entry__.build()")
    L = C.CDLL(str(path))
    P, i64, i32 = C.c_void_p, C.c_int64, C.c_int
    L.zd_build.restype = P
    L.zd_build.argtypes = [P, i64, i32]
    L.zd_build_ex.restype = P
    L.zd_build_ex.argtypes = [P, i64, i32, C.POINTER(_Opts)]
    L.zd_knn.restype = i32
    L.zd_knn.argtypes = [P, P, i64, i32, P, P]
    L.zd_knn_ex.restype = i32
    L.zd_knn_ex.argtypes = [P, P, i64, i32, P, P, i32]
    if hasattr(L, "zd_knn_range"):   # (older experiment builds lack the newer entry points)
        L.zd_knn_range.restype = i32
        L.zd_knn_range.argtypes = [P, i64, i64, i32, P, P, i32]
    L.zd_insert.restype = i64
    L.zd_insert.argtypes = [P, P, i64]
    L.zd_delete.restype = i64
    L.zd_delete.argtypes = [P, P, i64]
    L.zd_size.restype = i64
    L.zd_size.argtypes = [P]
    L.zd_live_ids.restype = i32
    L.zd_live_ids.argtypes = [P, P]
    L.zd_set_stream.restype = i32
    L.zd_set_stream.argtypes = [P, P]
    L.zd_free.restype = None
    L.zd_free.argtypes = [P]
    L.zd_last_error.restype = C.c_char_p
    L.zd_last_error.argtypes = []
    L.zd_last_error_code.restype = i32
    L.zd_last_error_code.argtypes = []
    L.zd_get_info.restype = i32
    L.zd_get_info.argtypes = [P, C.POINTER(_Info)]
    L.zd_export.restype = i32
    L.zd_export.argtypes = [P, P, P, P, P, P]
    L.zd_set_timing.restype = i32
    L.zd_set_timing.argtypes = [P, i32]
    if hasattr(L, "zd_trim"):
        L.zd_trim.restype = i32
        L.zd_trim.argtypes = []
    L.zd_kernel_launches.restype = i64
    L.zd_kernel_launches.argtypes = []
    L.zd_get_timing.restype = i32
    L.zd_get_timing.argtypes = [P, C.POINTER(C.c_float), i32]
    L.zd_knn_stats.restype = i32
    L.zd_knn_stats.argtypes = [P, i32, i32]
    _lib = L
    return L


def last_error() -> str:
    return load().zd_last_error().decode()


def _check(rc: int) -> int:
    if rc < 0:
        raise ZdError(rc, last_error())
    return rc


def _ptr(a) -> Optional[int]:
    """Raw pointer of a contiguous torch tensor / numpy array (None for None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if not a.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return a.data_ptr()


def _as_i32(a):
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=np.int32)
    import torch
    if a.dtype != torch.int32:
        a = a.to(torch.int32)
    return a.contiguous()


def _release_after(src, staged) -> None:
    """If marshalling made a temporary CUDA copy of the caller's array (dtype or
    layout conversion), wait for the device before the temporary can be freed: the
    library may still be reading it on the tree's stream when the call returns (torch's
    caching allocator would otherwise hand the memory to other work)."""
    if staged is not src and not isinstance(staged, np.ndarray) and staged is not None and staged.is_cuda:
        import torch
        torch.cuda.synchronize(staged.device)


def _current_stream() -> Optional[int]:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream().cuda_stream
    except Exception:
        pass
    return None


class ZdTree:
    """Handle to a device-resident zd-tree (wraps zd_tree*)."""

    def __init__(self, handle: int, dim: int):
        self._h = handle
        self.dim = dim

    # -- lifetime
    def zd_free(self):
        if self._h:
            load().zd_free(self._h)
            self._h = None

    close = zd_free

    def __del__(self):
        try:
            self.zd_free()
        except Exception:
            pass

    @property
    def handle(self) -> int:
        if not self._h:
            raise ZdError(ZD_EINVAL, "tree already freed")
        return self._h

    # -- queries
    def zd_knn(self, k: int, queries=None, out_idx=None, out_dist2=None, device=None, root_based: bool = False,
               warp: bool = False):
        """Exact k-NN.  queries=None: all live points (rows by ascending live id).
        Returns (out_idx int32 [m,k], out_dist2 int64 [m,k]); allocated on `device`
        (default: cuda) when not given.  root_based=True: the root-based search
        variant (zd_knn_ex, ZD_KNN_ROOT_BASED); warp=True: the large-k
        warp-per-query kernel for any k (ZD_KNN_WARP; always used for k > 32).  Same
        answer either way."""
        import torch
        q = None if queries is None else _as_i32(queries)
        m = self.zd_size() if q is None else int(q.shape[0])
        if out_idx is None:
            dev = device or "cuda"
            out_idx = torch.empty((m, k), dtype=torch.int32, device=dev)
            out_dist2 = torch.empty((m, k), dtype=torch.int64, device=dev)
        flags = (ZD_KNN_ROOT_BASED if root_based else 0) | (ZD_KNN_WARP if warp else 0)
        if flags:
            _check(load().zd_knn_ex(self.handle, _ptr(q), m, k, _ptr(out_idx), _ptr(out_dist2), flags))
        else:
            _check(load().zd_knn(self.handle, _ptr(q), m, k, _ptr(out_idx), _ptr(out_dist2)))
        _release_after(queries, q)
        return out_idx, out_dist2

    def zd_knn_range(self, k: int, pos_lo: int, pos_hi: int, out_idx, out_dist2, root_based: bool = False,
                     warp: bool = False):
        """All-points k-NN of the live points at sorted positions [pos_lo, pos_hi) only
        (one shard of the queries); writes their rows of the full
        [zd_size(), k] device outputs."""
        flags = (ZD_KNN_ROOT_BASED if root_based else 0) | (ZD_KNN_WARP if warp else 0)
        _check(load().zd_knn_range(self.handle, int(pos_lo), int(pos_hi), k, _ptr(out_idx), _ptr(out_dist2), flags))
        return out_idx, out_dist2

    def zd_insert(self, batch) -> int:
        b = _as_i32(batch)
        r = _check(load().zd_insert(self.handle, _ptr(b), int(b.shape[0])))
        _release_after(batch, b)
        return r

    def zd_delete(self, ids) -> int:
        i = _as_i32(ids)
        r = _check(load().zd_delete(self.handle, _ptr(i), int(i.shape[0])))
        _release_after(ids, i)
        return r

    def zd_size(self) -> int:
        return _check(load().zd_size(self.handle))

    def zd_live_ids(self, device=None):
        import torch
        out = torch.empty(self.zd_size(), dtype=torch.int32, device=device or "cuda")
        _check(load().zd_live_ids(self.handle, _ptr(out)))
        return out

    def zd_set_stream(self, stream) -> None:
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        _check(load().zd_set_stream(self.handle, s))

    # -- introspection
    def zd_get_info(self) -> dict:
        info = _Info()
        _check(load().zd_get_info(self.handle, C.byref(info)))
        out = {}
        for f, _ in _Info._fields_:
            v = getattr(info, f)
            out[f] = list(v) if isinstance(v, C.Array) else v
        return out

    def zd_export(self) -> dict:
        """Host copies of the sorted arrays and the node arrays (numpy)."""
        info = self.zd_get_info()
        n, nl, ni, w = info["n"], info["n_leaves"], info["n_internal"], info["node_words"]
        keys = np.empty(n, np.uint64)
        recs = np.empty((n, 4), np.int32)
        ls = np.empty(nl + 1, np.int32)
        lp = np.empty(nl, np.int32)
        nodes = np.empty((ni, w), np.int32)
        _check(load().zd_export(self.handle, _ptr(keys), _ptr(recs), _ptr(ls), _ptr(lp), _ptr(nodes)))
        return dict(info=info, keys=keys, recs=recs, leaf_start=ls, leaf_parent=lp, nodes=nodes)

    def zd_set_timing(self, enable: bool = True) -> None:
        _check(load().zd_set_timing(self.handle, int(enable)))

    def zd_get_timing(self) -> dict:
        buf = (C.c_float * len(PHASES))()
        c = _check(load().zd_get_timing(self.handle, buf, len(PHASES)))
        return {PHASES[i]: float(buf[i]) for i in range(c)}


KNN_STATS = ("packets", "queries", "nodes", "pops", "ascents", "spans", "passes", "candidates", "hits",
             "rounds", "compactions", "survivors", "survivors_max", "cycles", "max_packet", "deferred") + tuple(f"hist{i}" for i in range(32)) + (
    "insertions", "seed_hits", "seed_insertions", "seed_rounds", "lane_compactions", "need_pairs", "raw_staged")


def zd_knn_stats(reset: bool = True) -> dict:
    """Work counters of the k-NN kernel (profiling build only, ZD_LIB=stats)."""
    out = np.zeros(len(KNN_STATS), np.int64)
    n = _check(load().zd_knn_stats(_ptr(out), len(KNN_STATS), int(reset)))
    return dict(zip(KNN_STATS[:n], out[:n].tolist()))


def query_partition(n: int, parts: int, part: int, align: int = 32) -> tuple[int, int]:
    """Sorted-position range [lo, hi) of shard `part` of `parts` over n queries: equal
    contiguous Morton ranges, boundaries rounded to whole 32-query packets (so no
    packet straddles two shards); the ranges tile [0, n) exactly."""
    if parts < 1 or not 0 <= part < parts or n < 0:
        raise ValueError("need parts >= 1, 0 <= part < parts, n >= 0")

    def cut(r):   # nearest packet boundary to r/parts of the queries
        if r >= parts:
            return n
        return min(n, (2 * n * r + parts * align) // (2 * parts * align) * align)

    return cut(part), cut(part + 1)


def zd_trim() -> None:
    """Release the memory cached in the library's device pool (zd_trim)."""
    _check(load().zd_trim())


def zd_kernel_launches() -> int:
    """Process-wide number of CUDA kernels libzd.so has launched."""
    return int(load().zd_kernel_launches())


def zd_build(points, dim: Optional[int] = None, leaf_max: int = 16, stream=None, timing: bool = False,
             shift=None) -> ZdTree:
    """Build a zd-tree over int32 points [n, dim] (point i gets id i).  shift: the
    random shift of P:235 applied to every point (zd_opts.shift): 2D (sx, sy) in
    [0, 2^30); 3D (sx, sy, sz) in [0, 2^21)."""
    p = _as_i32(points)
    n = int(p.shape[0])
    dim = int(p.shape[1]) if dim is None else dim
    s = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    if s is None:
        s = _current_stream()
    sh = (C.c_int32 * 3)(*(list(shift) + [0] * (3 - len(shift)))) if shift is not None else (C.c_int32 * 3)()
    opts = _Opts(s, leaf_max, int(timing), int(shift is not None), sh)
    h = load().zd_build_ex(_ptr(p) if n else None, n, dim, C.byref(opts))
    _release_after(points, p)
    if not h:
        raise ZdError(load().zd_last_error_code(), last_error())
    return ZdTree(h, dim)


__all__ = ["zd_build", "zd_kernel_launches", "zd_trim", "query_partition", "zd_knn_stats", "ZdTree", "ZdError", "load", "build_lib", "last_error", "ZD_K_MAX", "ZD_KNN_WARP", "PHASES",
           "ZD_OK", "ZD_EINVAL", "ZD_ERANGE", "ZD_ENOMEM", "ZD_ECUDA"]
