"""Pins for the CPU oracle (-m "not gpu").

Each test ties the oracle to something other than itself: the paper's or
SPEC's worked examples (tests/golden/), closed forms, invariants, brute force
written independently with numpy, and Poisson-process statistics.
"""
import json
import math

import numpy as np
import pytest

import zdgen
from conftest import GOLDEN

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def _golden(name):
    return json.loads((GOLDEN / name).read_text())


# --------------------------------------------------------------- Morton keys

def test_morton_golden(oracle_mod):
    for ex in _golden("morton_examples.json")["examples"]:
        assert oracle_mod.key(ex["point"]) == ex["key"], ex["cite"]


@pytest.mark.parametrize("dim,B", [(2, 30), (3, 21)])
def test_morton_closed_forms(oracle_mod, dim, B):
    # P:187 + S:49: the top bit of axis a lands at key bit dim*B-1-a.
    for a in range(dim):
        p = [0] * dim
        p[a] = 1 << (B - 1)
        assert oracle_mod.key(p) == 1 << (dim * B - 1 - a)
        p[a] = 1  # lowest bit of axis a -> bit dim-1-a
        assert oracle_mod.key(p) == 1 << (dim - 1 - a)
    assert oracle_mod.key([(1 << B) - 1] * dim) == (1 << (dim * B)) - 1


@pytest.mark.parametrize("dim", [2, 3])
def test_morton_bit_conservation_and_injective(oracle_mod, dim):
    pts = zdgen.uniform(20000, dim, seed=11)
    k = oracle_mod.keys(pts)
    # interleaving permutes bits: popcount is conserved
    pc_pts = sum(np.array([bin(int(v)).count("1") for v in pts[:, a]]) for a in range(dim))
    pc_keys = np.array([bin(int(v)).count("1") for v in k])
    assert np.array_equal(pc_pts, pc_keys)
    # distinct coordinates -> distinct keys
    uniq_pts = np.unique(pts, axis=0).shape[0]
    assert np.unique(k).size == uniq_pts


@pytest.mark.parametrize("dim", [2, 3])
def test_morton_monotone_and_range_property(oracle_mod, dim):
    rng = np.random.default_rng(5)
    B = 30 if dim == 2 else 21
    lim = 1 << B
    for _ in range(2000):
        a = rng.integers(0, lim, size=dim)
        b = rng.integers(0, lim, size=dim)
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        c = lo + (rng.random(dim) * (hi - lo + 1)).astype(np.int64).clip(0, hi - lo)
        klo, khi, kc = oracle_mod.key(lo), oracle_mod.key(hi), oracle_mod.key(c)
        # points in the rectangle spanned by p and q fall between them
        assert klo <= kc <= khi
        # S:122 monotonicity in each coordinate
        ax = rng.integers(0, dim)
        if c[ax] + 1 < lim:
            c2 = c.copy()
            c2[ax] += 1
            assert oracle_mod.key(c2) > kc


def test_in_box(oracle_mod):
    assert oracle_mod.in_box(np.array([[0, (1 << 30) - 1]]))
    assert not oracle_mod.in_box(np.array([[0, 1 << 30]]))
    assert not oracle_mod.in_box(np.array([[-1, 0]]))
    assert oracle_mod.in_box(np.array([[0, 0, (1 << 21) - 1]]))
    assert not oracle_mod.in_box(np.array([[0, 0, 1 << 21]]))


# ---------------------------------------------------------------- geometry

def test_box_golden(oracle_mod):
    g = _golden("box_examples.json")
    for ex in g["boxd2"]:
        assert oracle_mod.boxd2(ex["q"], ex["lo"], ex["hi"]) == ex["d2"], ex["cite"]
    for ex in g["margin"]:
        assert oracle_mod.margin(ex["q"], ex["lo"], ex["hi"]) == ex["m"], ex["cite"]


def test_boxd2_brute(oracle_mod):
    # boxd2 = min over the box's lattice points of d^2 (brute force on tiny boxes)
    rng = np.random.default_rng(3)
    for _ in range(200):
        lo = rng.integers(0, 6, size=2)
        hi = lo + rng.integers(0, 4, size=2)
        q = rng.integers(0, 12, size=2)
        xs, ys = np.meshgrid(np.arange(lo[0], hi[0] + 1), np.arange(lo[1], hi[1] + 1))
        brute = int(((xs - q[0]) ** 2 + (ys - q[1]) ** 2).min())
        assert oracle_mod.boxd2(q, lo, hi) == brute


def test_nset_golden(oracle_mod):
    for ex in _golden("nset_examples.json")["examples"]:
        got = oracle_mod.nset_demo(ex["k"], ex["insert"])
        assert got == [tuple(r) for r in ex["result"]], ex["cite"]


# -------------------------------------------------------------------- tree

def check_tree_invariants(t, leaf_max=16):
    """Structural invariants of the canonical zd-tree (Alg. 1)."""
    keys, ids, _ = t.sorted_points()
    nd = t.nodes()
    n = t.n
    # sorted by (key, id), a permutation of the ids
    if n > 1:
        assert np.all((keys[1:] > keys[:-1]) | ((keys[1:] == keys[:-1]) & (ids[1:] > ids[:-1])))
    assert np.array_equal(np.sort(ids), np.sort(t.ids))
    split = nd["split"]
    leaves = np.nonzero(split < 0)[0]
    internal = np.nonzero(split >= 0)[0]
    assert len(internal) == max(len(leaves) - 1, 0)
    # every point in exactly one leaf
    cover = np.zeros(n, np.int64)
    for v in leaves:
        cover[nd["lo"][v]:nd["hi"][v]] += 1
    assert np.all(cover == 1)
    pts = np.zeros((n, 3), np.int64)
    _, _, coords = t.sorted_points()
    pts[:] = coords
    dim = t.dim
    for v in range(len(split)):
        lo, hi = nd["lo"][v], nd["hi"][v]
        if hi > lo:
            assert np.array_equal(nd["bmin"][v][:dim], pts[lo:hi, :dim].min(0))
            assert np.array_equal(nd["bmax"][v][:dim], pts[lo:hi, :dim].max(0))
        if split[v] < 0:
            assert hi - lo <= leaf_max or keys[lo] == keys[hi - 1]
        else:
            b = int(split[v])
            L, R = nd["left"][v], nd["right"][v]
            assert nd["parent"][L] == v and nd["parent"][R] == v
            assert nd["lo"][L] == lo and nd["hi"][R] == hi and nd["hi"][L] == nd["lo"][R]
            assert hi - lo > leaf_max and keys[lo] != keys[hi - 1]
            kk = keys[lo:hi]
            s = nd["hi"][L]
            # children partition the range by bit b ...
            assert np.all(((kk[: s - lo] >> np.uint64(b)) & np.uint64(1)) == 0)
            assert np.all(((kk[s - lo:] >> np.uint64(b)) & np.uint64(1)) == 1)
            # ... no empty cut: both sides non-empty, all keys share the bits above b
            assert lo < s < hi
            assert np.all((kk >> np.uint64(b + 1)) == (kk[0] >> np.uint64(b + 1)))
            for c in (L, R):
                if split[c] >= 0:
                    assert split[c] < b
    return nd


def test_tree_2x2_grid(oracle_mod):
    # d=2, leaf cutoff 1, 2x2 grid -> four leaves, depth 2, Morton order keys 0..3
    t = oracle_mod.Tree(np.array([[0, 0], [0, 1], [1, 0], [1, 1]]), leaf_max=1)
    nd = check_tree_invariants(t, leaf_max=1)
    assert (nd["split"] < 0).sum() == 4
    depth = 0
    v = int(np.nonzero(nd["split"] < 0)[0][0])
    while nd["parent"][v] >= 0:
        v = nd["parent"][v]
        depth += 1
    assert depth == 2
    assert list(t.sorted_points()[0]) == [0, 1, 2, 3]


def test_tree_tiny(oracle_mod):
    t = oracle_mod.Tree(np.zeros((0, 2), np.int32))   # S:187 empty -> single empty leaf
    nd = t.nodes()
    assert len(nd["split"]) == 1 and nd["split"][0] == -1
    t = oracle_mod.Tree(np.array([[5, 6, 7]]))          # S:189 one point -> single leaf
    nd = t.nodes()
    assert len(nd["split"]) == 1 and nd["split"][0] == -1 and nd["hi"][0] == 1


@pytest.mark.parametrize("dist,dim,n", [("uniform", 2, 5000), ("uniform", 3, 5000), ("plummer", 3, 5000),
                                        ("sphere", 3, 5000), ("dup", 3, 3000), ("dup", 2, 3000)])
def test_tree_invariants(oracle_mod, dist, dim, n):
    pts = zdgen.points(dist, n, dim, seed=21)
    check_tree_invariants(oracle_mod.Tree(pts))


def test_tree_depth_thm21(oracle_mod):
    # Thm 2.1: height O(log n).  Uniform 3D, 2^17 points: mean leaf depth
    # close to log2(n / mean leaf size), max within a few levels.
    pts = zdgen.uniform(1 << 17, 3, seed=9)
    t = oracle_mod.Tree(pts)
    nd = t.nodes()
    parent = nd["parent"]
    depth = np.zeros(len(parent), np.int64)
    for v in range(len(parent)):  # preorder: parent before child
        if parent[v] >= 0:
            depth[v] = depth[parent[v]] + 1
    leaves = nd["split"] < 0
    mean_leaf = (nd["hi"] - nd["lo"])[leaves].mean()
    assert 8 <= mean_leaf <= 16
    assert abs(depth[leaves].mean() - math.log2(t.n / mean_leaf)) < 1.5
    assert depth.max() <= math.log2(t.n) + 4


# --------------------------------------------------------------------- k-NN

def numpy_brute(points, qrows, k, ids=None):
    """Independent brute force: numpy distance row + lexsort by (d2, id)."""
    p = np.asarray(points, np.int64)
    ids = np.arange(len(p)) if ids is None else np.asarray(ids)
    oi = np.full((len(qrows), k), -1, np.int32)
    od = np.full((len(qrows), k), np.iinfo(np.int64).max, np.int64)
    for r, q in enumerate(qrows):
        d = ((p - p[q]) ** 2).sum(1)
        keep = ids != ids[q]
        order = np.lexsort((ids[keep], d[keep]))[:k]
        oi[r, :len(order)] = ids[keep][order]
        od[r, :len(order)] = d[keep][order]
    return oi, od


@pytest.mark.parametrize("dist,dim", [("uniform", 2), ("uniform", 3), ("dup", 2), ("plummer", 3)])
def test_brute_vs_numpy(oracle_mod, dist, dim):
    pts = zdgen.points(dist, 700, dim, seed=4)
    rows = np.arange(0, 700, 7)
    for k in (1, 5, 12, 128):
        oi, od = oracle_mod.brute_knn(pts, None, pts[rows], rows.astype(np.int32), k)
        ni, nd = numpy_brute(pts, rows, k)
        assert np.array_equal(oi, ni) and np.array_equal(od, nd)


def test_knn_golden(oracle_mod):
    for ex in _golden("knn_examples.json")["examples"]:
        pts = np.array(ex["points"], np.int32)
        t = oracle_mod.Tree(pts, leaf_max=1)
        for leaf_max in (1, 16):
            t = oracle_mod.Tree(pts, leaf_max=leaf_max)
            oi, od, _ = t.knn_all(ex["k"], nthreads=1)
            assert oi[ex["query"]].tolist() == ex["idx"], ex["cite"]
            assert od[ex["query"]].tolist() == ex["d2"], ex["cite"]


CASES = [("uniform", 2, 3000), ("uniform", 3, 3000), ("plummer", 3, 3000), ("sphere", 3, 3000), ("kuzmin", 2, 3000),
         ("dup", 3, 2000), ("dup", 2, 2000)]


@pytest.mark.parametrize("dist,dim,n", CASES)
@pytest.mark.parametrize("k", [1, 5, 10, 100, 128])
def test_tree_knn_equals_brute(oracle_mod, dist, dim, n, k):
    pts = zdgen.points(dist, n, dim, seed=17)
    t = oracle_mod.Tree(pts)
    oi, od, cnt = t.knn_all(k)
    ri, rd, _ = t.knn_all(k, root_based=True)
    rows = np.arange(n, dtype=np.int32)
    bi, bd = oracle_mod.brute_knn(pts, None, pts, rows, k)
    assert np.array_equal(oi, bi) and np.array_equal(od, bd)
    assert np.array_equal(ri, bi) and np.array_equal(rd, bd)
    assert cnt["dist_evals"] > 0


def test_lattice_all_rows(oracle_mod):
    # tie-heavy: 8^3 lattice and 16^2 lattice, every row vs brute force
    for side, dim in ((8, 3), (16, 2)):
        pts = zdgen.grid(side, dim)
        for leaf_max in (1, 4, 16):
            t = oracle_mod.Tree(pts, leaf_max=leaf_max)
            for k in (1, 6, 10, 27):
                oi, od, _ = t.knn_all(k)
                bi, bd = oracle_mod.brute_knn(pts, None, pts, np.arange(len(pts), dtype=np.int32), k)
                assert np.array_equal(oi, bi) and np.array_equal(od, bd)


def test_external_queries(oracle_mod):
    # NEXT-1: bit-based and root-based dynamic queries == brute force, no self-exclusion
    for dist, dim in (("uniform", 3), ("plummer", 3), ("uniform", 2), ("dup", 2)):
        pts = zdgen.points(dist, 3000, dim, seed=2)
        q = zdgen.points(dist if dist != "dup" else "uniform", 500, dim, seed=99)
        if dist == "dup":
            q = q % 8
        t = oracle_mod.Tree(pts)
        bi, bd = oracle_mod.brute_knn(pts, None, q, None, 10)
        for rb in (False, True):
            oi, od, _ = t.knn_queries(q, 10, root_based=rb)
            assert np.array_equal(oi, bi) and np.array_equal(od, bd)


def test_knn_row_invariants(oracle_mod):
    pts = zdgen.points("sphere", 20000, 3, seed=8)
    t = oracle_mod.Tree(pts)
    oi, od, _ = t.knn_all(10)
    n = len(pts)
    assert np.all((od[:, 1:] > od[:, :-1]) | ((od[:, 1:] == od[:, :-1]) & (oi[:, 1:] > oi[:, :-1])))
    assert not np.any(oi == np.arange(n)[:, None])          # self absent
    p = pts.astype(np.int64)
    d = ((p[oi] - p[:, None, :]) ** 2).sum(-1)               # d2 recomputed from coordinates
    assert np.array_equal(d, od)


def test_poisson_closed_form_2d(oracle_mod):
    # SURVEY §8(c) pins: 2D Poisson process, E[d2_k] = k / (pi rho).  C1 size.
    n, k = 65536, 10
    pts = zdgen.uniform(n, 2, seed=1)
    _, od, _ = oracle_mod.Tree(pts).knn_all(k)
    rho = n / float(1 << 60)
    for kk in (1, 10):
        expect = kk / (math.pi * rho)
        got = od[:, kk - 1].astype(np.float64).mean()
        assert abs(got / expect - 1) < 0.03, (kk, got, expect)


def test_poisson_closed_form_3d(oracle_mod):
    # 3D: E[d2_k] = (3/(4 pi rho))^(2/3) Gamma(k+2/3)/Gamma(k)
    n, k = 1 << 20, 10
    pts = zdgen.uniform(n, 3, seed=3)
    _, od, _ = oracle_mod.Tree(pts).knn_all(k)
    rho = n / float(1 << 63)
    for kk in (1, 10):
        expect = (3 / (4 * math.pi * rho)) ** (2 / 3) * math.gamma(kk + 2 / 3) / math.gamma(kk)
        got = od[:, kk - 1].astype(np.float64).mean()
        assert abs(got / expect - 1) < 0.03, (kk, got, expect)


# ------------------------------------------------------------------ updates

def test_update_inverse_and_equivalence(oracle_mod):
    base = zdgen.uniform(4000, 3, seed=6)
    live = oracle_mod.LiveSet(base)
    t0 = live.tree()
    r0 = t0.knn_all(10)
    batch = zdgen.uniform(700, 3, seed=7)
    first = live.insert(batch)
    assert first == 4000
    t1 = live.tree()
    # after insert == oracle build of the union with ids 4000..
    allp = np.concatenate([base, batch])
    bi, bd = oracle_mod.brute_knn(allp, None, allp, np.arange(len(allp), dtype=np.int32), 10)
    oi, od, _ = t1.knn_all(10)
    assert np.array_equal(oi, bi) and np.array_equal(od, bd)
    check_tree_invariants(t1)
    assert live.delete(np.arange(4000, 4700)) == 700
    assert live.delete(np.array([4000, -5, 99999])) == 0      # absent/dead ids skipped
    r1 = live.tree().knn_all(10)
    assert np.array_equal(r0[0], r1[0]) and np.array_equal(r0[1], r1[1])


def test_delete_rows_follow_live_ids(oracle_mod):
    base = zdgen.uniform(3000, 2, seed=12)
    live = oracle_mod.LiveSet(base)
    kill = zdgen.delete_ids(3000, 1000, seed=8)
    assert live.delete(kill) == 1000
    t = live.tree()
    oi, od, _ = t.knn_all(5)
    ids = live.live_ids()
    pts = base[ids]
    bi, bd = oracle_mod.brute_knn(pts, ids, pts, ids, 5)
    assert np.array_equal(oi, bi) and np.array_equal(od, bd)
    check_tree_invariants(t)


# ------------------------------------------------------------ random shift

SHIFTS = [(0, 0), (1, 2), ((1 << 30) - 1, (1 << 30) - 1), (123456789, 987654321 % (1 << 30))]


@pytest.mark.parametrize("shift", SHIFTS)
@pytest.mark.parametrize("dist", ["uniform", "dup", "kuzmin"])
def test_random_shift_pins(oracle_mod, dist, shift):
    """NEXT-4 random shift (Lemma 2.2), 2D: the tree of the shifted points
    is still a valid zd-tree (invariants), its keys are the 31-bit interleave of the
    shifted coordinates (independent big-int bit loop), and the k-NN answer is the
    translation-invariant plain definition: brute force on the unshifted points."""
    pts = zdgen.points(dist, 3000, 2, seed=5)
    t = oracle_mod.Tree(pts, shift=shift)
    check_tree_invariants(t)
    keys, ids, coords = t.sorted_points()
    sp = pts.astype(np.int64) + np.asarray(shift, np.int64)
    assert np.array_equal(coords[:, :2], sp[ids])
    for j in range(0, len(ids), 97):
        x, y = (int(v) for v in sp[ids[j]])
        key = 0
        for b in range(30, -1, -1):
            key = (key << 2) | (((x >> b) & 1) << 1) | ((y >> b) & 1)
        assert int(keys[j]) == key
    rows = np.arange(len(pts), dtype=np.int32)
    bi, bd = oracle_mod.brute_knn(pts, None, pts, rows, 10)
    oi, od, _ = t.knn_all(10)
    assert np.array_equal(oi, bi) and np.array_equal(od, bd)
    q = zdgen.uniform(400, 2, seed=6)
    qi, qd, _ = t.knn_queries(q, 7)
    bqi, bqd = oracle_mod.brute_knn(pts, None, q, None, 7)
    assert np.array_equal(qi, bqi) and np.array_equal(qd, bqd)


def test_random_shift_changes_the_tree(oracle_mod):
    # a shift that moves points across Morton cell boundaries changes the canonical tree
    pts = zdgen.uniform(4000, 2, seed=8)
    a, b = oracle_mod.Tree(pts), oracle_mod.Tree(pts, shift=(1 << 29, 12345))
    assert not np.array_equal(a.sorted_points()[1], b.sorted_points()[1])
    p3 = zdgen.uniform(4000, 3, seed=9)
    a, b = oracle_mod.Tree(p3), oracle_mod.Tree(p3, shift=(1 << 20, 777, 3))
    assert not np.array_equal(a.sorted_points()[1], b.sorted_points()[1])


# ---- work counters -----------------------------------
# dist = leaf points scanned (own point included), box = nodes entered by searchDown,
# ascents of searchUp, replacements = insertions into the k-best set (fills +
# evictions), evictions = insertions into a full set.  They set the roofline's
# algorithmic op count (bench.py), so they are pinned to a hand count and to App. A.

def test_counters_hand_counted_2x2_grid(oracle_mod):
    """2x2 grid, leaf size 1, k = 1 (the S:190 tree: four leaves under two nodes).
    Query (0,0) id 0: own leaf (1 scan, self), sibling leaf (0,1): 1 box + 1 scan
    (fill d2=1); ascent; margin test at the left node fails ((0+1)^2 = 1 is not > 1);
    right node entered (box d2 1 <= 1), its children by box distance: leaf (1,0)
    (1 box, 1 scan: (1, id 2) does not beat (1, id 0)), leaf (1,1) (1 box, pruned:
    2 > 1); ascent to the root.  -> 3 scans, 4 boxes, 2 ascents, 1 fill.  Queries id 1
    and id 3 mirror it; ids 2 and 3 end with an eviction each, because their first
    d2 = 1 neighbour (id 3 / id 2) loses the (d2, id) tie to one found later (id 0 /
    id 1).  Totals: 12 scans, 16 boxes, 8 ascents, 4 fills + 2 evictions."""
    pts = np.array([[0, 0], [0, 1], [1, 0], [1, 1]], np.int32)
    _, _, cnt = oracle_mod.Tree(pts, leaf_max=1).knn_all(1, nthreads=1)
    assert cnt == dict(dist_evals=12, box_tests=16, ascents=8, replacements=6, evictions=2)
    # two points: each query scans its own leaf, enters the sibling leaf, ascends once
    _, _, cnt = oracle_mod.Tree(np.array([[0, 0], [5, 0]], np.int32), leaf_max=1).knn_all(1, nthreads=1)
    assert cnt == dict(dist_evals=4, box_tests=2, ascents=2, replacements=2, evictions=0)


@pytest.mark.parametrize("dim,app_a", [
    (3, dict(dist_evals=91.0, box_tests=44.6, ascents=8.97, evictions=13.0, leaves=89_380)),
    (2, dict(dist_evals=43.8, box_tests=16.4, ascents=5.22, evictions=8.7, leaves=89_475)),
])
def test_counters_match_appendix_a(oracle_mod, dim, app_a):
    """Per-query work at n = 10^6 uniform, k = 10 against SURVEY App. A (its
    independent numpy model of the same search), within 3%; fills are exactly k."""
    pts = zdgen.uniform(1_000_000, dim, seed=3 if dim == 3 else 2)
    t = oracle_mod.Tree(pts)
    _, _, cnt = t.knn_all(10)
    per_q = {k: v / t.n for k, v in cnt.items()}
    for key in ("dist_evals", "box_tests", "ascents", "evictions"):
        assert abs(per_q[key] / app_a[key] - 1) < 0.03, (key, per_q[key], app_a[key])
    assert per_q["replacements"] - per_q["evictions"] == pytest.approx(10.0)
    leaves = int((t.nodes()["split"] < 0).sum())
    assert abs(leaves / app_a["leaves"] - 1) < 0.01


@pytest.mark.parametrize("dist", ["uniform", "plummer", "sphere"])
@pytest.mark.parametrize("shift", [(0, 0, 0), (1, 2, 3), (2**21 - 1, 12345, 2**20)])
def test_random_shift_3d_pins(oracle_mod, dist, shift):
    """NEXT-4 random shift in 3D (Lemma 2.2; reading R31): shifted
    coordinates take 22 bits; the key is the interleave of their levels 21..1 (63 bits,
    checked by an independent big-int bit loop), the tree stays a valid zd-tree over
    those keys, and the answer is the plain definition on the unshifted points."""
    pts = zdgen.points(dist, 3000, 3, seed=15)
    t = oracle_mod.Tree(pts, shift=shift)
    check_tree_invariants(t)
    keys, ids, coords = t.sorted_points()
    sp = pts.astype(np.int64) + np.asarray(shift, np.int64)
    assert np.array_equal(coords, sp[ids])
    assert int(sp.max()) < 2**22
    for j in range(0, len(ids), 89):
        x, y, z = (int(v) for v in sp[ids[j]])
        key = 0
        for b in range(21, 0, -1):
            key = (key << 3) | (((x >> b) & 1) << 2) | (((y >> b) & 1) << 1) | ((z >> b) & 1)
        assert int(keys[j]) == key
    rows = np.arange(len(pts), dtype=np.int32)
    bi, bd = oracle_mod.brute_knn(pts, None, pts, rows, 10)
    oi, od, _ = t.knn_all(10)
    assert np.array_equal(oi, bi) and np.array_equal(od, bd)
    q = zdgen.uniform(400, 3, seed=16)
    qi, qd, _ = t.knn_queries(q, 7)
    bqi, bqd = oracle_mod.brute_knn(pts, None, q, None, 7)
    assert np.array_equal(qi, bqi) and np.array_equal(qd, bqd)
