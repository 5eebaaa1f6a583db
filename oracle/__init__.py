"""CPU oracle for the zd-tree hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2111_04182_b200) never imports it and shares no code with it.

Thin ctypes wrapper over ``zd_oracle.c`` (plain C, sequential build, query loop
over host threads).  See the C file's header for the paper passages each
function follows.  Updates (reading 17) are done here by
rebuilding the canonical tree of the live set: insert appends the batch with
ids n_next, n_next+1, ... (reading 20); delete erases ids (reading 19).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_DIR = Path(__file__).resolve().parent
_SRC = _DIR / "zd_oracle.c"
_LIB = _DIR / "liboracle.so"

NCNT = 5
COUNTER_NAMES = ("dist_evals", "box_tests", "ascents", "replacements", "evictions")


def build_lib(force: bool = False) -> Path:
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["gcc", "-O2", "-g", "-std=c11", "-shared", "-fPIC", "-pthread",
                               str(_SRC), "-o", str(tmp)])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(str(build_lib()))
        P = C.c_void_p
        i64, i32 = C.c_int64, C.c_int
        L.orc_key.restype = C.c_uint64
        L.orc_key.argtypes = [P, i32]
        L.orc_keys.argtypes = [P, i64, i32, P]
        L.orc_in_box.argtypes = [P, i64, i32]
        L.orc_boxd2.restype = i64
        L.orc_boxd2.argtypes = [P, P, P, i32]
        L.orc_margin.restype = i64
        L.orc_margin.argtypes = [P, P, P, i32]
        L.orc_nset_demo.argtypes = [i32, P, P, i32, P, P]
        L.orc_build.restype = P
        L.orc_build.argtypes = [P, P, i64, i32, i32]
        L.orc_build_bits.restype = P
        L.orc_build_bits.argtypes = [P, P, i64, i32, i32, i32]
        L.orc_build_levels.restype = P
        L.orc_build_levels.argtypes = [P, P, i64, i32, i32, i32, i32]
        L.orc_free.argtypes = [P]
        L.orc_size.restype = i64
        L.orc_size.argtypes = [P]
        L.orc_num_nodes.restype = C.c_int32
        L.orc_num_nodes.argtypes = [P]
        L.orc_root.restype = C.c_int32
        L.orc_root.argtypes = [P]
        L.orc_export_points.argtypes = [P, P, P, P]
        L.orc_export_nodes.argtypes = [P, P, P, P, P]
        for f in (L.orc_knn_all, L.orc_knn_all_root):
            f.argtypes = [P, i32, i32, P, P, P]
        L.orc_knn_queries.argtypes = [P, P, i64, i32, i32, i32, P, P, P]
        L.orc_brute_knn.argtypes = [P, P, i64, i32, P, P, i64, i32, i32, P, P]
        L.orc_num_cores.restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def num_cores() -> int:
    return int(lib().orc_num_cores())


def keys(points: np.ndarray) -> np.ndarray:
    pts = _c32(points)
    n, dim = pts.shape
    out = np.empty(n, dtype=np.uint64)
    lib().orc_keys(_p(pts), n, dim, _p(out))
    return out


def key(point) -> int:
    p = _c32(point)
    return int(lib().orc_key(_p(p), p.shape[0]))


def in_box(points: np.ndarray) -> bool:
    pts = _c32(points)
    return bool(lib().orc_in_box(_p(pts), pts.shape[0], pts.shape[1]))


def boxd2(q, lo, hi) -> int:
    q, lo, hi = _c32(q), _c32(lo), _c32(hi)
    return int(lib().orc_boxd2(_p(q), _p(lo), _p(hi), q.shape[0]))


def margin(q, lo, hi) -> int:
    q, lo, hi = _c32(q), _c32(lo), _c32(hi)
    return int(lib().orc_margin(_p(q), _p(lo), _p(hi), q.shape[0]))


def nset_demo(k: int, pairs):
    """Insert (d2, id) pairs into an empty k-best set; returns the sorted set."""
    d = np.ascontiguousarray([p[0] for p in pairs], dtype=np.int64)
    i = np.ascontiguousarray([p[1] for p in pairs], dtype=np.int32)
    od = np.empty(k, np.int64)
    oi = np.empty(k, np.int32)
    cnt = lib().orc_nset_demo(k, _p(d), _p(i), len(pairs), _p(od), _p(oi))
    return [(int(od[j]), int(oi[j])) for j in range(cnt)]


class Tree:
    """Oracle zd-tree over (points, ids).

    shift: the random shift of P:235 ("select a random shift ... kept throughout"),
    added to every point (and query); the tree then stores the shifted coordinates.
    2D: (sx, sy) in [0, 2^30), keys of 31 bits per axis (62 bits).  3D: (sx, sy, sz)
    in [0, 2^21), shifted coordinates of 22 bits; the key interleaves their levels
    21 .. 1 (63 bits: the Morton order of the shifted grid at cell size 2; DESIGN
    reading R31)."""

    def __init__(self, points: np.ndarray, ids: np.ndarray | None = None, leaf_max: int = 16, shift=None):
        pts = _c32(points)
        self.shift = None if shift is None else np.asarray(shift, np.int64)[: pts.shape[1]]
        if self.shift is not None:
            pts = _c32((pts.astype(np.int64) + self.shift).astype(np.int32))
        self.points = pts
        self.n, self.dim = self.points.shape
        self.ids = np.arange(self.n, dtype=np.int32) if ids is None else _c32(ids)
        bits = (30 if self.dim == 2 else 21) + (1 if self.shift is not None else 0)
        lo = 1 if (self.shift is not None and self.dim == 3) else 0
        self._h = lib().orc_build_levels(_p(self.points), _p(self.ids), self.n, self.dim, leaf_max, bits, lo)
        if not self._h:
            raise ValueError("orc_build failed")
        self.leaf_max = leaf_max

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_free(h)
            self._h = None

    def sorted_points(self):
        """(keys u64[n], ids i32[n], coords i32[n,3]) in (key, id) order."""
        k = np.empty(self.n, np.uint64)
        i = np.empty(self.n, np.int32)
        c = np.empty((self.n, 3), np.int32)
        lib().orc_export_points(self._h, _p(k), _p(i), _p(c))
        return k, i, c

    def nodes(self) -> dict:
        nn = int(lib().orc_num_nodes(self._h))
        lohi = np.empty((nn, 2), np.int64)
        split = np.empty(nn, np.int32)
        links = np.empty((nn, 3), np.int32)
        bbox = np.empty((nn, 6), np.int32)
        lib().orc_export_nodes(self._h, _p(lohi), _p(split), _p(links), _p(bbox))
        return dict(lo=lohi[:, 0], hi=lohi[:, 1], split=split, parent=links[:, 0],
                    left=links[:, 1], right=links[:, 2], bmin=bbox[:, :3], bmax=bbox[:, 3:],
                    root=int(lib().orc_root(self._h)))

    def _run(self, fn, k, nthreads, m):
        oi = np.empty((m, k), np.int32)
        od = np.empty((m, k), np.int64)
        cnt = np.zeros(NCNT, np.int64)
        rc = fn(oi, od, cnt)
        if rc != 0:
            raise ValueError("oracle query failed")
        return oi, od, dict(zip(COUNTER_NAMES, cnt.tolist()))

    def knn_all(self, k: int, nthreads: int = 0, root_based: bool = False):
        """All-points k-NN (leaf-based Alg. 3, or root-based Alg. 2); rows by ascending id."""
        f = lib().orc_knn_all_root if root_based else lib().orc_knn_all
        return self._run(lambda oi, od, c: f(self._h, k, nthreads, _p(oi), _p(od), _p(c)), k, nthreads, self.n)

    def knn_queries(self, queries: np.ndarray, k: int, nthreads: int = 0, root_based: bool = False):
        q = _c32(queries)
        if self.shift is not None:
            q = _c32((q.astype(np.int64) + self.shift).astype(np.int32))
        m = q.shape[0]
        return self._run(lambda oi, od, c: lib().orc_knn_queries(
            self._h, _p(q), m, k, int(root_based), nthreads, _p(oi), _p(od), _p(c)), k, nthreads, m)


def brute_knn(points: np.ndarray, ids: np.ndarray | None, qpoints: np.ndarray,
              qids: np.ndarray | None, k: int, nthreads: int = 0):
    """Plain-definition k-NN by full scan (H3)."""
    pts = _c32(points)
    n, dim = pts.shape
    ids = None if ids is None else _c32(ids)
    qp = _c32(qpoints).reshape(-1, dim)
    qi = None if qids is None else _c32(qids)
    nq = qp.shape[0]
    oi = np.empty((nq, k), np.int32)
    od = np.empty((nq, k), np.int64)
    rc = lib().orc_brute_knn(_p(pts), _p(ids), n, dim, _p(qp), _p(qi), nq, k, nthreads, _p(oi), _p(od))
    if rc != 0:
        raise ValueError("brute force failed")
    return oi, od


class LiveSet:
    """Oracle of the batch-dynamic path: the canonical tree of the live multiset.

    insert(batch) appends with ids n_next..; delete(ids) erases present ids and
    returns how many were deleted (absent/dead/duplicate ids are skipped).
    """

    def __init__(self, points: np.ndarray, leaf_max: int = 16, shift=None):
        self.points = _c32(points)
        self.ids = np.arange(self.points.shape[0], dtype=np.int32)
        self.n_next = self.points.shape[0]
        self.leaf_max = leaf_max
        self.shift = shift

    def insert(self, batch: np.ndarray) -> int:
        b = _c32(batch)
        first = self.n_next
        self.points = np.concatenate([self.points, b.reshape(-1, self.points.shape[1])])
        self.ids = np.concatenate([self.ids, np.arange(first, first + b.shape[0], dtype=np.int32)])
        self.n_next += b.shape[0]
        return first

    def delete(self, ids: np.ndarray) -> int:
        kill = np.isin(self.ids, np.asarray(ids, dtype=np.int32))
        self.points = self.points[~kill]
        self.ids = self.ids[~kill]
        return int(kill.sum())

    def tree(self) -> Tree:
        return Tree(self.points, self.ids, self.leaf_max, shift=self.shift)

    def live_ids(self) -> np.ndarray:
        return np.sort(self.ids)
