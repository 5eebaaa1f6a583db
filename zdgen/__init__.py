"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the zd-tree's arithmetic (no Morton keys, no tree,
no distances).  It only draws integer grid coordinates and id selections, so
both sides of every parity test consume byte-identical int32 arrays
(SURVEY.md §8(c) items 23-26).

RNG: counter-based SplitMix64 output function.
  word(seed, point i, draw j) = mix64(seed * G2 + (i * 64 + j + 1) * G)
with G = 0x9E3779B97F4A7C15 (the SplitMix64 increment) and G2 a second odd
constant that separates seeds.  Output is independent of thread count and of
how many points are drawn.

Distributions (PAPER.md P:1212 names them; the grid mapping is ours):
  uniform2d  : top 30 bits per axis -> [0, 2^30)^2          (configs C1, C2)
  uniform3d  : top 21 bits per axis -> [0, 2^21)^3          (C3, C5)
  plummer    : r = 1/sqrt(u^(-2/3) - 1), u in (0,1) open; reject+redraw if
               r > 50; isotropic direction z = 2v-1, phi = 2*pi*w;
               grid = min(2^21-1, floor((x + 50)/100 * 2^21))      (C4a)
  sphere     : unit sphere (z = 2v-1, phi = 2*pi*w);
               grid = min(2^21-1, floor((x + 1) * 2^20))          (C4b)
  kuzmin     : 2D Kuzmin disk, R = sqrt((1-u)^-2 - 1), reject R > 100, angle 2*pi*w;
               grid = min(2^30-1, floor((x + 100)/200 * 2^30))    (paper's 5th set)
  delete ids : the m ids in [0, n) with the smallest (mix64(seed, id), id)
"""
from __future__ import annotations

import numpy as np

_G = np.uint64(0x9E3779B97F4A7C15)
_G2 = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
DRAWS_PER_POINT = 64  # counter stride per point; Plummer uses 3 per attempt

B2, B3 = 30, 21  # bits per axis: fixed universe box


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def words(seed: int, idx: np.ndarray, draw) -> np.ndarray:
    """SplitMix64 word for (seed, point idx, draw index)."""
    idx = np.asarray(idx, dtype=np.uint64)
    draw = np.asarray(draw, dtype=np.uint64)
    with np.errstate(over="ignore"):
        ctr = idx * np.uint64(DRAWS_PER_POINT) + draw + np.uint64(1)
        z = np.uint64(seed) * _G2 + ctr * _G
    return _mix64(z)


def _unit_open(w: np.ndarray) -> np.ndarray:
    """Top 53 bits * 2^-53 + 2^-54: uniform on the open interval (0, 1)."""
    return (w >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) + 2.0 ** -54


def _unit(w: np.ndarray) -> np.ndarray:
    return (w >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform(n: int, dim: int, seed: int, first_index: int = 0) -> np.ndarray:
    """n x dim int32, i.i.d. uniform on [0, 2^B)^dim (B = 30 in 2D, 21 in 3D)."""
    B = B2 if dim == 2 else B3
    idx = np.arange(first_index, first_index + n, dtype=np.uint64)
    out = np.empty((n, dim), dtype=np.int32)
    for a in range(dim):
        out[:, a] = (words(seed, idx, a) >> np.uint64(64 - B)).astype(np.int32)
    return out


def _direction(v: np.ndarray, w: np.ndarray):
    z = 2.0 * v - 1.0
    phi = 2.0 * np.pi * w
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return s * np.cos(phi), s * np.sin(phi), z


def plummer(n: int, seed: int, rmax: float = 50.0) -> np.ndarray:
    """n x 3 int32 Plummer-model points quantised to [0, 2^21)^3."""
    idx = np.arange(n, dtype=np.uint64)
    r = np.full(n, np.nan)
    vv = np.empty(n)
    ww = np.empty(n)
    todo = np.arange(n)
    attempt = 0
    while todo.size:
        if 3 * attempt + 2 >= DRAWS_PER_POINT:
            raise RuntimeError("plummer: rejection budget exhausted")
        ii = idx[todo]
        u = _unit_open(words(seed, ii, 3 * attempt))
        v = _unit(words(seed, ii, 3 * attempt + 1))
        w = _unit(words(seed, ii, 3 * attempt + 2))
        rr = 1.0 / np.sqrt(u ** (-2.0 / 3.0) - 1.0)
        ok = rr <= rmax
        sel = todo[ok]
        r[sel], vv[sel], ww[sel] = rr[ok], v[ok], w[ok]
        todo = todo[~ok]
        attempt += 1
    dx, dy, dz = _direction(vv, ww)
    out = np.empty((n, 3), dtype=np.int32)
    scale = float(1 << B3)
    for a, c in enumerate((dx * r, dy * r, dz * r)):
        g = np.floor((c + rmax) / (2.0 * rmax) * scale)
        out[:, a] = np.clip(g, 0, (1 << B3) - 1).astype(np.int32)
    return out


def sphere(n: int, seed: int) -> np.ndarray:
    """n x 3 int32 points uniform on the unit sphere, quantised to [0, 2^21)^3."""
    idx = np.arange(n, dtype=np.uint64)
    v = _unit(words(seed, idx, 0))
    w = _unit(words(seed, idx, 1))
    dx, dy, dz = _direction(v, w)
    out = np.empty((n, 3), dtype=np.int32)
    for a, c in enumerate((dx, dy, dz)):
        g = np.floor((c + 1.0) * float(1 << (B3 - 1)))
        out[:, a] = np.clip(g, 0, (1 << B3) - 1).astype(np.int32)
    return out


def kuzmin(n: int, seed: int, rmax: float = 100.0) -> np.ndarray:
    """n x 2 int32 points of a Kuzmin disk (the paper's 2DKuzmin), surface
    density proportional to (1 + R^2)^(-3/2): M(<R) = 1 - 1/sqrt(1 + R^2), so
    R = sqrt((1 - u)^(-2) - 1) for u in (0,1) open; reject + redraw R > rmax; angle
    phi = 2*pi*w; grid = min(2^30-1, floor((x + rmax)/(2 rmax) * 2^30)) per axis."""
    idx = np.arange(n, dtype=np.uint64)
    r = np.full(n, np.nan)
    ww = np.empty(n)
    todo = np.arange(n)
    attempt = 0
    while todo.size:
        if 2 * attempt + 1 >= DRAWS_PER_POINT:
            raise RuntimeError("kuzmin: rejection budget exhausted")
        ii = idx[todo]
        u = _unit_open(words(seed, ii, 2 * attempt))
        w = _unit(words(seed, ii, 2 * attempt + 1))
        rr = np.sqrt((1.0 - u) ** -2.0 - 1.0)
        ok = rr <= rmax
        sel = todo[ok]
        r[sel], ww[sel] = rr[ok], w[ok]
        todo = todo[~ok]
        attempt += 1
    phi = 2.0 * np.pi * ww
    out = np.empty((n, 2), dtype=np.int32)
    scale = float(1 << B2)
    for a, c in enumerate((r * np.cos(phi), r * np.sin(phi))):
        g = np.floor((c + rmax) / (2.0 * rmax) * scale)
        out[:, a] = np.clip(g, 0, (1 << B2) - 1).astype(np.int32)
    return out


def delete_ids(n: int, m: int, seed: int) -> np.ndarray:
    """The m ids of [0, n) with the smallest (mix64 word, id); int32, ascending id."""
    if m >= n:
        return np.arange(n, dtype=np.int32)
    idx = np.arange(n, dtype=np.uint64)
    h = words(seed, idx, 0)
    part = np.argpartition(h, m)[: m + 1]
    # exact (h, id) order on the candidate boundary
    order = np.lexsort((part, h[part]))
    chosen = part[order[:m]]
    # resolve a possible tie on h at the boundary against ids outside `part`
    hmax = h[chosen].max()
    if (h == hmax).sum() > (h[chosen] == hmax).sum():
        cand = np.nonzero(h <= hmax)[0]
        order = np.lexsort((cand, h[cand]))
        chosen = cand[order[:m]]
    return np.sort(chosen).astype(np.int32)


def grid(side: int, dim: int) -> np.ndarray:
    """All points of the tie-heavy lattice [0, side)^dim (row-major), int32."""
    ax = np.arange(side, dtype=np.int32)
    mesh = np.meshgrid(*([ax] * dim), indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=1).astype(np.int32)


def duplicates(n: int, dim: int, seed: int, side: int = 8) -> np.ndarray:
    """n points drawn uniformly from a tiny [0, side)^dim lattice: many coincident points."""
    idx = np.arange(n, dtype=np.uint64)
    out = np.empty((n, dim), dtype=np.int32)
    for a in range(dim):
        out[:, a] = (words(seed, idx, a) % np.uint64(side)).astype(np.int32)
    return out


# The five BASELINE.json configs (SURVEY §8(d) seeds).
CONFIGS = {
    "C1": dict(dim=2, n=65_536, dist="uniform", seed=1),
    "C2": dict(dim=2, n=10_000_000, dist="uniform", seed=2),
    "C3": dict(dim=3, n=10_000_000, dist="uniform", seed=3),
    "C4a": dict(dim=3, n=10_000_000, dist="plummer", seed=4),
    "C4b": dict(dim=3, n=10_000_000, dist="sphere", seed=5),
    "K2": dict(dim=2, n=10_000_000, dist="kuzmin", seed=9),   # not a BASELINE config: P:1212's 2DKuzmin
    "C5": dict(dim=3, n=10_000_000, dist="uniform", seed=6,
               insert_m=1_000_000, insert_seed=7, delete_m=1_000_000, delete_seed=8),
}


def points(dist: str, n: int, dim: int, seed: int) -> np.ndarray:
    if dist == "uniform":
        return uniform(n, dim, seed)
    if dist == "plummer":
        assert dim == 3
        return plummer(n, seed)
    if dist == "sphere":
        assert dim == 3
        return sphere(n, seed)
    if dist == "kuzmin":
        assert dim == 2
        return kuzmin(n, seed)
    if dist == "dup":
        return duplicates(n, dim, seed)
    raise ValueError(dist)


def config_points(name: str, n: int | None = None) -> np.ndarray:
    c = CONFIGS[name]
    return points(c["dist"], c["n"] if n is None else n, c["dim"], c["seed"])


def insert_batch(m: int, dim: int, seed: int) -> np.ndarray:
    return uniform(m, dim, seed)
