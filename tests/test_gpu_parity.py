"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Sizes span several sort tiles (3328 keys), several topology tiles (2048 pairs) and
ragged tails; edge cases cover empty / single / duplicate-heavy inputs, every k
template and leaf sizes 1..32.
"""
import numpy as np
import pytest
import torch

import zdgen
from parity_util import assert_same_structure, first_row_mismatch

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_knn_all(tree, k):
    oi, od = tree.zd_knn(k)
    torch.cuda.synchronize()
    return oi.cpu().numpy(), od.cpu().numpy()


def check_rows(gi, gd, oi, od):
    bad = first_row_mismatch(gi, gd, oi, od)
    assert bad.size == 0, f"{bad.size} rows differ, first row {bad[0]}: gpu {gi[bad[0]]} {gd[bad[0]]} oracle {oi[bad[0]]} {od[bad[0]]}"


# sort tiles of 3328 keys, one-pass topology tiles of 2048 pairs (n - 1 pairs)
SIZES = [0, 1, 2, 3, 16, 17, 33, 1000, 2047, 2048, 2049, 2050, 2815, 2816, 2817, 3327, 3328, 3329, 4097, 4098,
         6145, 6657, 20011]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dim", [2, 3])
def test_sort_and_structure_sizes(zd, oracle_mod, n, dim):
    pts = zdgen.uniform(n, dim, seed=100 + n)
    t = zd.zd_build(dev(pts))
    assert_same_structure(t.zd_export(), oracle_mod.Tree(pts))
    assert t.zd_size() == n


@pytest.mark.parametrize("n", [127, 128, 129, 130, 255, 256, 257, 383, 384, 385, 1153])
@pytest.mark.parametrize("dim", [2, 3])
def test_bottom_up_window_boundaries(zd, oracle_mod, n, dim):
    """leaf_max = 1 makes every point a leaf, so the leaf count sits on and around the
    bottom-up pass's 128-leaf windows: window-local nodes (written from shared memory
    after the block barrier) and window-crossing nodes (device-scope arrivals) must
    give the oracle's tree; the k-NN reads the nodes' point ranges, the delete fast
    path their leaf bounds."""
    pts = zdgen.uniform(n, dim, seed=900 + n)
    t = zd.zd_build(dev(pts), leaf_max=1)
    ot = oracle_mod.Tree(pts, leaf_max=1)
    assert_same_structure(t.zd_export(), ot)
    gi, gd = gpu_knn_all(t, 3)
    oi, od, _ = ot.knn_all(3)
    check_rows(gi, gd, oi, od)
    kill = np.array([n // 2], np.int32)
    assert t.zd_delete(dev(kill)) == 1
    live = oracle_mod.LiveSet(pts, leaf_max=1)
    live.delete(kill)
    assert_same_structure(t.zd_export(), live.tree())


@pytest.mark.parametrize("dist,dim", [("uniform", 2), ("uniform", 3), ("plummer", 3), ("sphere", 3),
                                      ("dup", 2), ("dup", 3)])
@pytest.mark.parametrize("leaf_max", [1, 4, 16, 32])
def test_structure_distributions(zd, oracle_mod, dist, dim, leaf_max):
    pts = zdgen.points(dist, 30000, dim, seed=7)
    t = zd.zd_build(dev(pts), leaf_max=leaf_max)
    assert_same_structure(t.zd_export(), oracle_mod.Tree(pts, leaf_max=leaf_max))


@pytest.mark.parametrize("dist,dim", [("uniform", 2), ("uniform", 3), ("plummer", 3), ("sphere", 3),
                                      ("kuzmin", 2), ("dup", 2), ("dup", 3)])
@pytest.mark.parametrize("k", [1, 3, 5, 10, 16, 32])
def test_knn_all_distributions(zd, oracle_mod, dist, dim, k):
    pts = zdgen.points(dist, 20000, dim, seed=11)
    t = zd.zd_build(dev(pts))
    gi, gd = gpu_knn_all(t, k)
    oi, od, _ = oracle_mod.Tree(pts).knn_all(k)
    check_rows(gi, gd, oi, od)


@pytest.mark.parametrize("leaf_max", [1, 2, 7, 16, 32])
def test_knn_leaf_sizes(zd, oracle_mod, leaf_max):
    pts = zdgen.points("plummer", 15000, 3, seed=3)
    t = zd.zd_build(dev(pts), leaf_max=leaf_max)
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = oracle_mod.Tree(pts).knn_all(10)
    check_rows(gi, gd, oi, od)


@pytest.mark.parametrize("n", [0, 1, 2, 5, 11, 17])
def test_knn_tiny_padding(zd, oracle_mod, n):
    pts = zdgen.uniform(n, 3, seed=n)
    t = zd.zd_build(dev(pts))
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = oracle_mod.Tree(pts).knn_all(10)
    check_rows(gi, gd, oi, od)
    if n:
        assert np.all(gi[:, max(n - 1, 0):] == -1)


def test_lattices_every_row(zd, oracle_mod):
    for side, dim in ((8, 3), (16, 2), (32, 2)):
        pts = zdgen.grid(side, dim)
        for k in (1, 6, 27):
            t = zd.zd_build(dev(pts))
            gi, gd = gpu_knn_all(t, k)
            bi, bd = oracle_mod.brute_knn(pts, None, pts, np.arange(len(pts), dtype=np.int32), k)
            check_rows(gi, gd, bi, bd)


def _far_corner_points(dim, seed):
    """Fine lattices and near-ties at the top of the universe box, where fp32 cannot
    represent 2D coordinates (ulp 64 at 2^30): exercises the fp32 prefilter's bound
    (knn.cu filter_bound) against exact int64 distances and (d2, id) ties."""
    B = 30 if dim == 2 else 21
    top = (1 << B) - 1
    rng = np.random.default_rng(seed)
    g = zdgen.grid(12, dim).astype(np.int64) * 3            # lattice spacing 3
    parts = [top - g,                                         # lattice in the far corner
             top - rng.integers(0, 40, size=(3000, dim)),     # dense cloud, many ties
             top - rng.integers(0, 1 << (B - 2), size=(3000, dim)),
             rng.integers(0, 1 << B, size=(3000, dim)),
             np.full((5, dim), top)]                          # coincident points
    return np.ascontiguousarray(np.concatenate(parts).astype(np.int32))


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("k", [1, 10, 32])
def test_knn_far_corner_ties(zd, oracle_mod, dim, k):
    pts = _far_corner_points(dim, seed=dim * 100 + k)
    t = zd.zd_build(dev(pts))
    gi, gd = gpu_knn_all(t, k)
    bi, bd = oracle_mod.brute_knn(pts, None, pts, np.arange(len(pts), dtype=np.int32), k)
    check_rows(gi, gd, bi, bd)


def test_c1_full_vs_brute_force(zd, oracle_mod):
    """Config C1 (65,536 2D uniform, seed 1): every row vs plain brute force."""
    pts = zdgen.config_points("C1")
    t = zd.zd_build(dev(pts))
    gi, gd = gpu_knn_all(t, 10)
    bi, bd = oracle_mod.brute_knn(pts, None, pts, np.arange(len(pts), dtype=np.int32), 10)
    check_rows(gi, gd, bi, bd)
    assert_same_structure(t.zd_export(), oracle_mod.Tree(pts))


def test_host_pointers_and_host_outputs(zd, oracle_mod):
    """The C ABI accepts host arrays (staged internally) and host outputs."""
    pts = zdgen.uniform(5000, 3, seed=5)
    t = zd.zd_build(pts)                      # numpy host array
    oi = np.empty((5000, 10), np.int32)
    od = np.empty((5000, 10), np.int64)
    t.zd_knn(10, out_idx=oi, out_dist2=od)     # host outputs, synchronous
    ri, rd, _ = oracle_mod.Tree(pts).knn_all(10)
    check_rows(oi, od, ri, rd)


@pytest.mark.parametrize("dist,dim", [("uniform", 3), ("plummer", 3), ("uniform", 2), ("dup", 2)])
@pytest.mark.parametrize("k", [1, 10, 32])
def test_external_queries(zd, oracle_mod, dist, dim, k):
    pts = zdgen.points(dist, 20000, dim, seed=21)
    q = zdgen.uniform(3000, dim, seed=22)
    if dist == "dup":
        q = q % 8
    if dist == "plummer":
        q = np.concatenate([q, zdgen.plummer(3000, 23)])
    t = zd.zd_build(dev(pts))
    gi, gd = t.zd_knn(k, queries=dev(q))
    torch.cuda.synchronize()
    bi, bd = oracle_mod.brute_knn(pts, None, q, None, k)
    check_rows(gi.cpu().numpy(), gd.cpu().numpy(), bi, bd)
    oi, od, _ = oracle_mod.Tree(pts).knn_queries(q, k)
    check_rows(gi.cpu().numpy(), gd.cpu().numpy(), oi, od)


def test_external_queries_empty_tree(zd):
    t = zd.zd_build(dev(np.zeros((0, 3), np.int32)))
    gi, gd = t.zd_knn(4, queries=dev(np.array([[1, 2, 3]], np.int32)))
    assert gi.cpu().tolist() == [[-1] * 4]
    assert gd.cpu().tolist() == [[np.iinfo(np.int64).max] * 4]


# ------------------------------------------------------------------ updates

@pytest.mark.parametrize("dim", [2, 3])
def test_insert_then_delete(zd, oracle_mod, dim):
    base = zdgen.uniform(30000, dim, seed=31)
    batch = zdgen.uniform(7000, dim, seed=32)
    t = zd.zd_build(dev(base))
    live = oracle_mod.LiveSet(base)
    r0 = gpu_knn_all(t, 10)
    first = t.zd_insert(dev(batch))
    assert first == live.insert(batch) == 30000
    assert t.zd_size() == 37000
    assert_same_structure(t.zd_export(), live.tree())
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = live.tree().knn_all(10)
    check_rows(gi, gd, oi, od)
    # delete the batch: every original row is restored bit-exactly
    assert t.zd_delete(dev(np.arange(30000, 37000, dtype=np.int32))) == 7000
    r1 = gpu_knn_all(t, 10)
    assert np.array_equal(r0[0], r1[0]) and np.array_equal(r0[1], r1[1])


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("n", [1, 2, 3, 9, 15, 16, 17])
def test_insert_delete_tiny_trees(zd, oracle_mod, dim, n):
    """Updates of trees that are a single leaf (2..16 points) or barely more: the
    insert fast path must refuse them cleanly (the located leaf of a
    single-leaf tree was left unwritten) and the result is the canonical tree."""
    base = zdgen.uniform(n, dim, seed=900 + n)
    t = zd.zd_build(dev(base))
    live = oracle_mod.LiveSet(base)
    for m, seed in ((1, 1), (2, 2), (5, 3)):
        batch = zdgen.uniform(m, dim, seed=950 + 10 * n + seed)
        assert t.zd_insert(dev(batch)) == live.insert(batch)
        assert_same_structure(t.zd_export(), live.tree())
        gi, gd = gpu_knn_all(t, 4)
        oi, od, _ = live.tree().knn_all(4)
        check_rows(gi, gd, oi, od)
    kill = np.array([0, n + 1, n + 100], dtype=np.int32)
    assert t.zd_delete(dev(kill)) == live.delete(kill)
    assert_same_structure(t.zd_export(), live.tree())


def test_delete_rows_and_live_ids(zd, oracle_mod):
    base = zdgen.uniform(40000, 3, seed=41)
    t = zd.zd_build(dev(base))
    live = oracle_mod.LiveSet(base)
    kill = zdgen.delete_ids(40000, 9000, seed=8)
    dup = np.concatenate([kill, kill[:100], np.array([-1, 40000, 10 ** 9], np.int32)])
    assert t.zd_delete(dev(dup)) == 9000 == live.delete(kill)
    assert t.zd_delete(dev(kill[:10])) == 0           # already dead: skipped
    assert np.array_equal(t.zd_live_ids().cpu().numpy(), live.live_ids())
    assert_same_structure(t.zd_export(), live.tree())
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = live.tree().knn_all(10)
    check_rows(gi, gd, oi, od)


def test_update_sequence_mixed(zd, oracle_mod):
    """Several rounds of insert / delete (C5 shape, small) stay canonical and exact."""
    rng = np.random.default_rng(4)
    base = zdgen.plummer(20000, 51)
    t = zd.zd_build(dev(base))
    live = oracle_mod.LiveSet(base)
    for r in range(6):
        b = zdgen.plummer(int(rng.integers(1, 5000)), 60 + r)
        assert t.zd_insert(dev(b)) == live.insert(b)
        ids = live.live_ids()
        kill = rng.choice(ids, size=min(len(ids), int(rng.integers(0, 6000))), replace=False).astype(np.int32)
        assert t.zd_delete(dev(kill)) == live.delete(kill)
        assert t.zd_size() == len(live.ids)
    assert_same_structure(t.zd_export(), live.tree())
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = live.tree().knn_all(10)
    check_rows(gi, gd, oi, od)


def test_insert_growth_and_delete_all(zd, oracle_mod):
    base = zdgen.uniform(100, 2, seed=1)
    t = zd.zd_build(dev(base))
    live = oracle_mod.LiveSet(base)
    for r in range(4):                                   # grows capacity several times
        b = zdgen.uniform(300 * (r + 1), 2, seed=70 + r)
        assert t.zd_insert(dev(b)) == live.insert(b)
    assert_same_structure(t.zd_export(), live.tree())
    assert t.zd_delete(dev(live.live_ids())) == len(live.ids)
    assert t.zd_size() == 0
    gi, gd = gpu_knn_all(t, 3)
    assert gi.shape == (0, 3)
    b = zdgen.uniform(50, 2, seed=99)
    first = t.zd_insert(dev(b))
    assert first == 100 + sum(300 * (r + 1) for r in range(4))


# ------------------------------------------------------------------- errors

def test_errors(zd):
    bad = np.array([[0, 1 << 21, 5]], np.int32)
    with pytest.raises(zd.ZdError) as e:
        zd.zd_build(dev(bad))
    assert e.value.code == zd.ZD_ERANGE
    with pytest.raises(zd.ZdError) as e:
        zd.zd_build(dev(np.array([[-1, 0]], np.int32)))
    assert e.value.code == zd.ZD_ERANGE
    pts = zdgen.uniform(1000, 3, seed=2)
    t = zd.zd_build(dev(pts))
    before = t.zd_export()
    with pytest.raises(zd.ZdError) as e:
        t.zd_insert(dev(np.concatenate([zdgen.uniform(10, 3, seed=3), bad])))
    assert e.value.code == zd.ZD_ERANGE
    after = t.zd_export()                            # all-or-nothing: unchanged
    assert np.array_equal(before["recs"], after["recs"]) and t.zd_size() == 1000
    assert t.zd_insert(dev(zdgen.uniform(1, 3, seed=4))) == 1000   # ids not consumed by the failed insert
    for k in (0, zd.ZD_K_MAX + 1):
        with pytest.raises(zd.ZdError) as e:
            t.zd_knn(k)
        assert e.value.code == zd.ZD_EINVAL
    with pytest.raises(zd.ZdError):
        t.zd_knn(5, queries=dev(bad))
    with pytest.raises(zd.ZdError):
        zd.zd_build(dev(pts), leaf_max=33)


def test_streams_and_timing(zd, oracle_mod):
    pts = zdgen.uniform(50000, 3, seed=9)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        t = zd.zd_build(dev(pts), stream=s)
        t.zd_set_timing(True)
        oi, od = t.zd_knn(10)
    s.synchronize()
    tm = t.zd_get_timing()
    assert tm["knn"] > 0
    ri, rd, _ = oracle_mod.Tree(pts).knn_all(10)
    check_rows(oi.cpu().numpy(), od.cpu().numpy(), ri, rd)


@pytest.mark.parametrize("mode", ["none", "all"])
@pytest.mark.parametrize("dist,dim", [("uniform", 2), ("uniform", 3), ("plummer", 3), ("sphere", 3), ("dup", 3)])
def test_knn_deferral_modes(zd, oracle_mod, monkeypatch, mode, dist, dim):
    """The k-NN kernel's second pass (packets deferred as incoherent, searched one query
    per warp) and the single-pass path both give the oracle's rows: ZD_KNN_DEFER=all
    sends every packet through the second pass, =none disables it."""
    monkeypatch.setenv("ZD_KNN_DEFER", mode)
    pts = zdgen.points(dist, 12000, dim, seed=21)
    t = zd.zd_build(dev(pts))
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = oracle_mod.Tree(pts).knn_all(10)
    check_rows(gi, gd, oi, od)
    q = zdgen.uniform(3000, dim, seed=22)
    qi, qd = t.zd_knn(10, queries=dev(q))
    torch.cuda.synchronize()
    oqi, oqd, _ = oracle_mod.Tree(pts).knn_queries(q, 10)
    check_rows(qi.cpu().numpy(), qd.cpu().numpy(), oqi, oqd)


@pytest.mark.parametrize("dist,dim", [("uniform", 2), ("uniform", 3), ("plummer", 3), ("sphere", 3), ("dup", 3)])
def test_knn_root_based(zd, oracle_mod, dist, dim):
    """Root-based search (zd_knn_ex ZD_KNN_ROOT_BASED) gives the same unique
    answer as the leaf-based search and the oracle, all-points and external queries."""
    pts = zdgen.points(dist, 9000, dim, seed=31)
    t = zd.zd_build(dev(pts))
    gi, gd = t.zd_knn(10, root_based=True)
    torch.cuda.synchronize()
    oi, od, _ = oracle_mod.Tree(pts).knn_all(10, root_based=True)
    check_rows(gi.cpu().numpy(), gd.cpu().numpy(), oi, od)
    q = zdgen.uniform(2000, dim, seed=32)
    qi, qd = t.zd_knn(10, queries=dev(q), root_based=True)
    torch.cuda.synchronize()
    oqi, oqd, _ = oracle_mod.Tree(pts).knn_queries(q, 10)
    check_rows(qi.cpu().numpy(), qd.cpu().numpy(), oqi, oqd)


# ------------------------------------------------- large k (warp-per-query kernel)

@pytest.mark.parametrize("dist,dim", [("uniform", 2), ("uniform", 3), ("plummer", 3), ("sphere", 3),
                                      ("kuzmin", 2), ("dup", 2), ("dup", 3)])
@pytest.mark.parametrize("k", [33, 64, 100, 128])
def test_knn_large_k(zd, oracle_mod, dist, dim, k):
    """k > 32 runs the warp-per-query kernel (knn_warp.cu; P:543's large-k container)."""
    pts = zdgen.points(dist, 6000, dim, seed=13)
    t = zd.zd_build(dev(pts))
    gi, gd = gpu_knn_all(t, k)
    oi, od, _ = oracle_mod.Tree(pts).knn_all(k)
    check_rows(gi, gd, oi, od)


@pytest.mark.parametrize("n", [0, 1, 2, 3, 16, 17, 33, 1000, 5633])
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("k", [1, 10, 32])
def test_knn_warp_forced_sizes(zd, oracle_mod, n, dim, k):
    """The warp kernel forced for small k (ZD_KNN_WARP) on tiny and ragged sizes."""
    pts = zdgen.uniform(n, dim, seed=200 + n)
    t = zd.zd_build(dev(pts))
    gi, gd = t.zd_knn(k, warp=True)
    torch.cuda.synchronize()
    oi, od, _ = oracle_mod.Tree(pts).knn_all(k)
    check_rows(gi.cpu().numpy(), gd.cpu().numpy(), oi, od)


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("k", [10, 100])
def test_knn_warp_far_corner_ties(zd, oracle_mod, dim, k):
    pts = _far_corner_points(dim, seed=dim * 1000 + k)
    t = zd.zd_build(dev(pts))
    gi, gd = t.zd_knn(k, warp=True)
    torch.cuda.synchronize()
    bi, bd = oracle_mod.brute_knn(pts, None, pts, np.arange(len(pts), dtype=np.int32), k)
    check_rows(gi.cpu().numpy(), gd.cpu().numpy(), bi, bd)


@pytest.mark.parametrize("dim", [2, 3])
def test_knn_warp_massive_ties(zd, oracle_mod, dim):
    """400 coincident copies of each of 6 sites: more equal distances than the warp
    kernel's buffer holds, so the exact (d2, id) tie resolution runs."""
    sites = zdgen.uniform(6, dim, seed=5)
    pts = np.ascontiguousarray(np.repeat(sites, 400, axis=0))
    t = zd.zd_build(dev(pts))
    for k in (100, 128):
        gi, gd = gpu_knn_all(t, k)
        bi, bd = oracle_mod.brute_knn(pts, None, pts, np.arange(len(pts), dtype=np.int32), k)
        check_rows(gi, gd, bi, bd)


def test_knn_warp_lattice_every_row(zd, oracle_mod):
    for side, dim in ((8, 3), (24, 2)):
        pts = zdgen.grid(side, dim)
        t = zd.zd_build(dev(pts))
        for k in (57, 125):
            gi, gd = gpu_knn_all(t, k)
            bi, bd = oracle_mod.brute_knn(pts, None, pts, np.arange(len(pts), dtype=np.int32), k)
            check_rows(gi, gd, bi, bd)


@pytest.mark.parametrize("dist,dim", [("uniform", 3), ("plummer", 3), ("uniform", 2), ("dup", 2)])
@pytest.mark.parametrize("k,warp", [(10, True), (64, False), (128, False)])
def test_knn_warp_external_and_root(zd, oracle_mod, dist, dim, k, warp):
    pts = zdgen.points(dist, 8000, dim, seed=41)
    q = zdgen.uniform(1500, dim, seed=42)
    if dist == "dup":
        q = q % 8
    t = zd.zd_build(dev(pts))
    gi, gd = t.zd_knn(k, queries=dev(q), warp=warp)
    torch.cuda.synchronize()
    bi, bd = oracle_mod.brute_knn(pts, None, q, None, k)
    check_rows(gi.cpu().numpy(), gd.cpu().numpy(), bi, bd)
    ri, rd = t.zd_knn(k, root_based=True, warp=warp)
    torch.cuda.synchronize()
    oi, od, _ = oracle_mod.Tree(pts).knn_all(k)
    check_rows(ri.cpu().numpy(), rd.cpu().numpy(), oi, od)


def test_knn_warp_after_updates(zd, oracle_mod):
    base = zdgen.plummer(15000, 61)
    t = zd.zd_build(dev(base))
    live = oracle_mod.LiveSet(base)
    b = zdgen.plummer(4000, 62)
    assert t.zd_insert(dev(b)) == live.insert(b)
    kill = zdgen.delete_ids(15000, 5000, seed=63)
    assert t.zd_delete(dev(kill)) == live.delete(kill)
    for k in (50, 128):
        gi, gd = gpu_knn_all(t, k)
        oi, od, _ = live.tree().knn_all(k)
        check_rows(gi, gd, oi, od)


# --------------------------------------- node buffers sized from the node count

@pytest.mark.parametrize("leaf_max", [1, 16])
@pytest.mark.parametrize("dist,dim", [("uniform", 3), ("plummer", 3), ("uniform", 2), ("dup", 3)])
def test_count_sized_node_buffers(zd, oracle_mod, monkeypatch, leaf_max, dist, dim):
    """Above ZD_EXACT_NODES_MIN points (2^25 by default) the node-indexed tree buffers
    are sized from each build's node count (one sync after the flag scan, growth when a
    rebuild has more nodes).  Threshold 0 runs that path at test sizes; leaf size 1
    forces the buffers to grow from the initial n/8 guess."""
    monkeypatch.setenv("ZD_EXACT_NODES_MIN", "0")
    pts = zdgen.points(dist, 9000, dim, seed=71)
    t = zd.zd_build(dev(pts), leaf_max=leaf_max)
    live = oracle_mod.LiveSet(pts, leaf_max=leaf_max)
    assert_same_structure(t.zd_export(), live.tree())
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = live.tree().knn_all(10)
    check_rows(gi, gd, oi, od)
    b = zdgen.points(dist, 4000, dim, seed=72)
    assert t.zd_insert(dev(b)) == live.insert(b)
    kill = zdgen.delete_ids(9000, 3000, seed=73)
    assert t.zd_delete(dev(kill)) == live.delete(kill)
    assert_same_structure(t.zd_export(), live.tree())
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = live.tree().knn_all(10)
    check_rows(gi, gd, oi, od)
    for n in (0, 1, 2, 17):
        small = zdgen.uniform(n, dim, seed=n)
        ts = zd.zd_build(dev(small), leaf_max=leaf_max)
        assert_same_structure(ts.zd_export(), oracle_mod.Tree(small, leaf_max=leaf_max))


# ------------------------------------------------------ random shift, 2D

SHIFTS = [(0, 0), (1, 2), ((1 << 30) - 1, (1 << 30) - 1), (123456789, 987654321 % (1 << 30))]


@pytest.mark.parametrize("shift", SHIFTS)
@pytest.mark.parametrize("dist,leaf_max", [("uniform", 16), ("dup", 16), ("kuzmin", 16), ("uniform", 1)])
def test_random_shift(zd, oracle_mod, dist, leaf_max, shift):
    """zd_opts.shift: the canonical tree of the shifted points (oracle with the same
    shift), and k-NN answers identical to the unshifted tree's (a translation)."""
    pts = zdgen.points(dist, 12000, 2, seed=81)
    t = zd.zd_build(dev(pts), leaf_max=leaf_max, shift=shift)
    assert t.zd_get_info()["shift"][:2] == list(shift)
    live = oracle_mod.LiveSet(pts, leaf_max=leaf_max, shift=shift)
    assert_same_structure(t.zd_export(), live.tree())
    u = zd.zd_build(dev(pts), leaf_max=leaf_max)
    for k in (10, 50):
        gi, gd = gpu_knn_all(t, k)
        ui, ud = gpu_knn_all(u, k)
        assert np.array_equal(gi, ui) and np.array_equal(gd, ud)
    oi, od, _ = live.tree().knn_all(10)
    check_rows(*gpu_knn_all(t, 10), oi, od)
    q = zdgen.uniform(2000, 2, seed=82)
    qi, qd = t.zd_knn(10, queries=dev(q))
    torch.cuda.synchronize()
    bi, bd = oracle_mod.brute_knn(pts, None, q, None, 10)
    check_rows(qi.cpu().numpy(), qd.cpu().numpy(), bi, bd)
    # updates keep the shift
    b = zdgen.points(dist, 3000, 2, seed=83)
    assert t.zd_insert(dev(b)) == live.insert(b)
    kill = zdgen.delete_ids(12000, 4000, seed=84)
    assert t.zd_delete(dev(kill)) == live.delete(kill)
    assert_same_structure(t.zd_export(), live.tree())
    oi, od, _ = live.tree().knn_all(10)
    check_rows(*gpu_knn_all(t, 10), oi, od)


SHIFTS3 = [(0, 0, 0), (1, 2, 3), ((1 << 21) - 1, (1 << 21) - 1, (1 << 21) - 1), (1234567, 7654, 1 << 20)]


@pytest.mark.parametrize("shift", SHIFTS3)
@pytest.mark.parametrize("dist,leaf_max", [("uniform", 16), ("plummer", 16), ("sphere", 16), ("dup", 16),
                                           ("uniform", 1)])
def test_random_shift_3d(zd, oracle_mod, dist, leaf_max, shift):
    """3D random shift (reading R31): the canonical tree over the keys of the
    shifted coordinates' levels 21..1 equals the oracle's, and every answer equals the
    unshifted tree's (a translation), for all-points, external queries and updates
    (fast and full paths)."""
    pts = zdgen.points(dist, 12000, 3, seed=85)
    t = zd.zd_build(dev(pts), leaf_max=leaf_max, shift=shift)
    assert t.zd_get_info()["shift"] == list(shift)
    live = oracle_mod.LiveSet(pts, leaf_max=leaf_max, shift=shift)
    assert_same_structure(t.zd_export(), live.tree())
    u = zd.zd_build(dev(pts), leaf_max=leaf_max)
    for k in (10, 50):
        gi, gd = gpu_knn_all(t, k)
        ui, ud = gpu_knn_all(u, k)
        assert np.array_equal(gi, ui) and np.array_equal(gd, ud)
    q = zdgen.uniform(2000, 3, seed=86)
    qi, qd = t.zd_knn(10, queries=dev(q))
    torch.cuda.synchronize()
    bi, bd = oracle_mod.brute_knn(pts, None, q, None, 10)
    check_rows(qi.cpu().numpy(), qd.cpu().numpy(), bi, bd)
    for m, seed in ((3, 87), (3000, 88)):   # a small (fast-path candidate) and a large batch
        b = zdgen.points(dist, m, 3, seed=seed)
        assert t.zd_insert(dev(b)) == live.insert(b)
        assert_same_structure(t.zd_export(), live.tree())
    kill = zdgen.delete_ids(12000, 4000, seed=89)
    assert t.zd_delete(dev(kill)) == live.delete(kill)
    assert_same_structure(t.zd_export(), live.tree())
    oi, od, _ = live.tree().knn_all(10)
    check_rows(*gpu_knn_all(t, 10), oi, od)


def test_random_shift_errors(zd):
    for bad in ((-1, 0, 0), (0, 1 << 21, 0)):
        with pytest.raises(zd.ZdError) as e:
            zd.zd_build(dev(zdgen.uniform(100, 3, seed=1)), shift=bad)
        assert e.value.code == zd.ZD_EINVAL
    for bad in ((-1, 0), (0, 1 << 30)):
        with pytest.raises(zd.ZdError) as e:
            zd.zd_build(dev(zdgen.uniform(100, 2, seed=1)), shift=bad)
        assert e.value.code == zd.ZD_EINVAL
    # the range check applies to the unshifted coordinates
    t = zd.zd_build(dev(zdgen.uniform(100, 2, seed=1)), shift=(5, 5))
    with pytest.raises(zd.ZdError) as e:
        t.zd_insert(dev(np.array([[1 << 30, 0]], np.int32)))
    assert e.value.code == zd.ZD_ERANGE


# ------------------------------------------------------------- adversarial inputs

def _adversarial(kind, dim):
    B = 30 if dim == 2 else 21
    top = (1 << B) - 1
    rng = np.random.default_rng(17)
    if kind == "deep":
        # one point per power of two on every axis: each split peels off one point, so
        # with leaf size 1 the canonical tree reaches depth ~dim*B (the 64-level bound)
        pts = [np.zeros(dim, np.int64)]
        for a in range(dim):
            for j in range(B):
                p = np.zeros(dim, np.int64)
                p[a] = 1 << j
                pts.append(p)
                q = np.full(dim, top, np.int64)
                q[a] = top - (1 << j)
                pts.append(q)
        return np.array(pts, np.int32)
    if kind == "collinear":
        x = rng.integers(0, 1 << B, size=4000)
        return np.stack([x] + [np.full(4000, 12345)] * (dim - 1), axis=1).astype(np.int32)
    if kind == "two_corners":
        a = rng.integers(0, 64, size=(3000, dim))
        return np.concatenate([a, top - a]).astype(np.int32)
    if kind == "one_site_plus_outliers":
        a = np.full((3000, dim), 777)
        b = rng.integers(0, 1 << B, size=(20, dim))
        return np.concatenate([a, b]).astype(np.int32)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["deep", "collinear", "two_corners", "one_site_plus_outliers"])
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("leaf_max", [1, 16])
def test_adversarial_inputs(zd, oracle_mod, kind, dim, leaf_max):
    pts = _adversarial(kind, dim)
    t = zd.zd_build(dev(pts), leaf_max=leaf_max)
    assert_same_structure(t.zd_export(), oracle_mod.Tree(pts, leaf_max=leaf_max))
    rows = np.arange(len(pts), dtype=np.int32)
    for k, warp in ((1, False), (10, False), (10, True), (100, False)):
        gi, gd = t.zd_knn(k, warp=warp)
        torch.cuda.synchronize()
        bi, bd = oracle_mod.brute_knn(pts, None, pts, rows, k)
        check_rows(gi.cpu().numpy(), gd.cpu().numpy(), bi, bd)
    q = _adversarial(kind, dim)[::3]
    gi, gd = t.zd_knn(10, queries=dev(q))
    torch.cuda.synchronize()
    bi, bd = oracle_mod.brute_knn(pts, None, q, None, 10)
    check_rows(gi.cpu().numpy(), gd.cpu().numpy(), bi, bd)
    if dim == 2:
        s = zd.zd_build(dev(pts), leaf_max=leaf_max, shift=(1 << 29, 3))
        gi, gd = s.zd_knn(10)
        torch.cuda.synchronize()
        bi, bd = oracle_mod.brute_knn(pts, None, pts, rows, 10)
        check_rows(gi.cpu().numpy(), gd.cpu().numpy(), bi, bd)


# ------------------------------------------- NEXT-2: insert fast path (incr.cu)

def _fitting_batch(t, pts, per_leaf, perturb, seed):
    """Points placed in leaves with spare room: copies of a leaf's point, optionally
    with the lowest coordinate bit flipped (stays in the leaf's Morton cell)."""
    ex = t.zd_export()
    ls = ex["leaf_start"]
    sizes = np.diff(ls)
    rng = np.random.default_rng(seed)
    leaves = np.nonzero(sizes <= 16 - per_leaf)[0]
    leaves = rng.choice(leaves, size=min(len(leaves), 300), replace=False)
    out = []
    for l in leaves:
        rec = ex["recs"][ls[l]]
        for _ in range(per_leaf):
            p = rec[:pts.shape[1]].astype(np.int64).copy()
            if perturb:
                p[rng.integers(0, pts.shape[1])] ^= 1
            out.append(p)
    return np.array(out, np.int32)


@pytest.mark.parametrize("dist,dim", [("uniform", 3), ("plummer", 3), ("uniform", 2), ("kuzmin", 2)])
@pytest.mark.parametrize("perturb", [False, True])
def test_insert_fast_path(zd, oracle_mod, monkeypatch, dist, dim, perturb):
    monkeypatch.delenv("ZD_INCR", raising=False)
    pts = zdgen.points(dist, 40000, dim, seed=91)
    t = zd.zd_build(dev(pts))
    live = oracle_mod.LiveSet(pts)
    fast0 = t.zd_get_info()["fast_inserts"]
    for r in range(3):   # first insert grows the capacity, later ones do not
        b = _fitting_batch(t, pts, 1 + r % 2, perturb, seed=r)
        assert t.zd_insert(dev(b)) == live.insert(b)
        assert_same_structure(t.zd_export(), live.tree())
    info = t.zd_get_info()
    assert info["fast_inserts"] - fast0 >= 2, "the fitting batches should take the fast path"
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = live.tree().knn_all(10)
    check_rows(gi, gd, oi, od)
    # a random batch overflows leaves: full rebuild, still canonical
    b = zdgen.points(dist, 3000, dim, seed=95)
    before = t.zd_get_info()["fast_inserts"]
    assert t.zd_insert(dev(b)) == live.insert(b)
    assert t.zd_get_info()["fast_inserts"] == before
    assert_same_structure(t.zd_export(), live.tree())
    # after a delete (topology rebuilt) the fast path applies again
    kill = zdgen.delete_ids(40000, 500, seed=96)
    assert t.zd_delete(dev(kill)) == live.delete(kill)
    b = _fitting_batch(t, pts, 1, perturb, seed=97)
    assert t.zd_insert(dev(b)) == live.insert(b)
    assert_same_structure(t.zd_export(), live.tree())
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = live.tree().knn_all(10)
    check_rows(gi, gd, oi, od)
    q = zdgen.uniform(1000, dim, seed=98)
    qi, qd = t.zd_knn(16, queries=dev(q))
    torch.cuda.synchronize()
    oqi, oqd, _ = live.tree().knn_queries(q, 16)
    check_rows(qi.cpu().numpy(), qd.cpu().numpy(), oqi, oqd)


def test_insert_fast_path_disabled_and_shifted(zd, oracle_mod, monkeypatch):
    pts = zdgen.uniform(30000, 2, seed=92)
    monkeypatch.setenv("ZD_INCR", "0")
    t = zd.zd_build(dev(pts))
    b = _fitting_batch(t, pts, 1, True, seed=1)
    t.zd_insert(dev(b))
    assert t.zd_get_info()["fast_inserts"] == 0
    monkeypatch.delenv("ZD_INCR")
    s = zd.zd_build(dev(pts), shift=(123457, 1 << 29))
    live = oracle_mod.LiveSet(pts, shift=(123457, 1 << 29))
    b = _fitting_batch(s, pts, 1, False, seed=2) - np.array([123457, 1 << 29], np.int32)   # unshift
    assert s.zd_insert(dev(b)) == live.insert(b)
    assert s.zd_get_info()["fast_inserts"] == 1
    assert_same_structure(s.zd_export(), live.tree())
    oi, od, _ = live.tree().knn_all(10)
    check_rows(*gpu_knn_all(s, 10), oi, od)


@pytest.mark.parametrize("dist,dim", [("uniform", 3), ("plummer", 3), ("uniform", 2), ("kuzmin", 2)])
def test_delete_fast_path(zd, oracle_mod, monkeypatch, dist, dim):
    """Deletes that keep the topology (no leaf emptied, every internal node keeps more
    than leaf_max points) shift positions and refit the dirty paths' boxes instead of
    rebuilding: removing points added by a fitting insert restores the original tree."""
    monkeypatch.delenv("ZD_INCR", raising=False)
    pts = zdgen.points(dist, 40000, dim, seed=93)
    t = zd.zd_build(dev(pts))
    live = oracle_mod.LiveSet(pts)
    before = t.zd_export()
    b = _fitting_batch(t, pts, 1, True, seed=11)
    first = t.zd_insert(dev(b))
    assert first == live.insert(b)
    new_ids = np.arange(first, first + len(b), dtype=np.int32)
    d0 = t.zd_get_info()["fast_deletes"]
    for part in np.array_split(new_ids, 3):
        assert t.zd_delete(dev(part)) == live.delete(part) == len(part)
        assert_same_structure(t.zd_export(), live.tree())
    assert t.zd_get_info()["fast_deletes"] - d0 == 3
    after = t.zd_export()
    assert np.array_equal(after["nodes"], before["nodes"]) and np.array_equal(after["leaf_start"], before["leaf_start"])
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = live.tree().knn_all(10)
    check_rows(gi, gd, oi, od)
    # single random deletes: fast or rebuilt, always canonical
    rng = np.random.default_rng(3)
    for r in range(6):
        kill = rng.choice(live.live_ids(), size=1 + r % 3, replace=False).astype(np.int32)
        assert t.zd_delete(dev(kill)) == live.delete(kill)
        assert_same_structure(t.zd_export(), live.tree())
    # a batch that empties nodes falls back to the rebuild
    kill = live.live_ids()[:3000].astype(np.int32)
    f = t.zd_get_info()["fast_deletes"]
    assert t.zd_delete(dev(kill)) == live.delete(kill)
    assert t.zd_get_info()["fast_deletes"] == f
    assert_same_structure(t.zd_export(), live.tree())
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = live.tree().knn_all(10)
    check_rows(gi, gd, oi, od)


def test_concurrent_handles_on_streams(zd, oracle_mod):
    """Different handles used at the same time from two host threads, each on its own
    CUDA stream with host input and output buffers (bench.py's pipelined e2e): build,
    insert, delete and the all-points query of each equal the oracle's, and a tree built
    on a second stream answers like one built on the default stream."""
    import threading
    from concurrent.futures import ThreadPoolExecutor
    cases = []
    for j in range(2):
        base = zdgen.uniform(20000 + 1000 * j, 3, seed=70 + j)
        batch = zdgen.uniform(1500, 3, seed=72 + j)
        kill = zdgen.delete_ids(len(base), 900, seed=74 + j)
        live = oracle_mod.LiveSet(base)
        live.insert(batch)
        live.delete(kill)
        oi, od, _ = live.tree().knn_all(10)
        cases.append((base, batch, kill, oi, od))
    streams = [torch.cuda.Stream() for _ in range(2)]
    lock = threading.Lock()

    def run(j):
        base, batch, kill, oi, od = cases[j]
        with torch.cuda.stream(streams[j]):
            for _ in range(3):
                t = zd.zd_build(base, stream=streams[j])      # host input (staged)
                t.zd_insert(batch)
                t.zd_delete(kill)
                gi = np.empty((t.zd_size(), 10), np.int32)
                gd = np.empty((t.zd_size(), 10), np.int64)
                t.zd_knn(10, out_idx=gi, out_dist2=gd)          # host output: synchronous
                t.zd_free()
                with lock:
                    check_rows(gi, gd, oi, od)
        return True

    with ThreadPoolExecutor(2) as ex:
        assert all(ex.map(run, range(2)))


def test_concurrent_knn_one_handle(zd, oracle_mod):
    """zd_knn is re-entrant on one handle ("queries can be conducted in
    parallel"): two host threads query the same tree, after updates (row map) and with
    timing on (per-call events), and both get the oracle's rows."""
    import threading
    base = zdgen.uniform(30000, 3, seed=61)
    t = zd.zd_build(dev(base))
    live = oracle_mod.LiveSet(base)
    batch = zdgen.uniform(3000, 3, seed=62)
    t.zd_insert(dev(batch)); live.insert(batch)
    kill = zdgen.delete_ids(30000, 2000, seed=63)
    t.zd_delete(dev(kill)); live.delete(kill)
    t.zd_set_timing(True)
    oi, od, _ = live.tree().knn_all(10)
    qs = zdgen.uniform(5000, 3, seed=64)
    qi, qd, _ = live.tree().knn_queries(qs, 5)
    errors = []

    def worker(external):
        try:
            for _ in range(6):
                if external:
                    gi, gd = t.zd_knn(5, queries=dev(qs))
                    torch.cuda.synchronize()
                    check_rows(gi.cpu().numpy(), gd.cpu().numpy(), qi, qd)
                else:
                    gi, gd = gpu_knn_all(t, 10)
                    check_rows(gi, gd, oi, od)
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(e)

    th = [threading.Thread(target=worker, args=(x,)) for x in (False, True, False)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors[0]
    assert t.zd_get_timing()["knn"] > 0


def test_trim_releases_pool(zd):
    t = zd.zd_build(dev(zdgen.uniform(200000, 3, seed=65)))
    t.zd_free()
    assert zd.load().zd_trim() == 0
    t = zd.zd_build(dev(zdgen.uniform(1000, 3, seed=66)))   # the pool grows again on demand
    assert t.zd_size() == 1000


@pytest.mark.parametrize("parts", [1, 3, 8])
def test_knn_range_shards(zd, oracle_mod, parts):
    """zd_knn_range (SURVEY §8(e) query shards): the shards' rows together equal the
    all-points answer, and each call leaves the other rows untouched; also after a
    delete (row map) and at k > 32 (warp kernel)."""
    base = zdgen.uniform(20011, 3, seed=71)
    t = zd.zd_build(dev(base))
    t.zd_delete(dev(zdgen.delete_ids(20011, 1000, seed=72)))
    n = t.zd_size()
    for k in (10, 40):
        ref_i, ref_d = gpu_knn_all(t, k)
        oi = torch.full((n, k), -7, dtype=torch.int32, device="cuda")
        od = torch.full((n, k), -7, dtype=torch.int64, device="cuda")
        seen = np.zeros(n, bool)
        for r in range(parts):
            lo, hi = zd.query_partition(n, parts, r)
            before = oi.cpu().numpy().copy()
            t.zd_knn_range(k, lo, hi, oi, od)
            torch.cuda.synchronize()
            after = oi.cpu().numpy()
            changed = np.any(after != before, axis=1)
            assert not np.any(changed & seen), "a shard rewrote another shard's rows"
            assert changed.sum() == hi - lo
            seen |= changed
        assert seen.all()
        assert np.array_equal(oi.cpu().numpy(), ref_i) and np.array_equal(od.cpu().numpy(), ref_d)
    with pytest.raises(zd.ZdError):
        t.zd_knn_range(10, 5, n + 1, oi, od)


@pytest.mark.parametrize("n", [1025, 2049, 4097, 10241])
def test_pt_leaf_covers_every_position(zd, oracle_mod, n):
    """Sizes with n - 1 a multiple of the topology tile (1024 pairs): the leaf of the
    last sorted position is written too (it seeds the last k-NN packet)."""
    pts = zdgen.uniform(n, 3, seed=n)
    t = zd.zd_build(dev(pts))
    ex = t.zd_export()
    ls = ex["leaf_start"]
    assert ls[-1] == n
    gi, gd = gpu_knn_all(t, 10)
    oi, od, _ = oracle_mod.Tree(pts).knn_all(10)
    check_rows(gi, gd, oi, od)


def test_converted_inputs(zd, oracle_mod):
    """int64 / non-contiguous CUDA inputs are converted by the binding into temporaries
    that stay alive until the device is done with them."""
    base = zdgen.uniform(5000, 3, seed=91)
    t = zd.zd_build(dev(base).to(torch.int64))
    live = oracle_mod.LiveSet(base)
    b = zdgen.uniform(4000, 3, seed=92)
    wide = torch.zeros((4000, 6), dtype=torch.int32, device="cuda")
    wide[:, ::2] = dev(b)
    assert t.zd_insert(wide[:, ::2]) == live.insert(b)              # non-contiguous view
    kill = zdgen.delete_ids(5000, 700, seed=93)
    assert t.zd_delete(dev(kill).to(torch.int64)) == live.delete(kill)
    q = zdgen.uniform(300, 3, seed=94)
    qi, qd = t.zd_knn(5, queries=dev(q).to(torch.int64))
    torch.cuda.synchronize()
    ot = live.tree()
    ei, ed, _ = ot.knn_queries(q, 5)
    check_rows(qi.cpu().numpy(), qd.cpu().numpy(), ei, ed)
    oi, od, _ = ot.knn_all(10)
    check_rows(*gpu_knn_all(t, 10), oi, od)


@pytest.mark.parametrize("dist,dim,shift", [("uniform", 3, None), ("uniform", 2, None), ("plummer", 3, None),
                                            ("sphere", 3, None), ("dup", 3, None), ("cube", 3, None),
                                            ("uniform", 3, (12345, 1 << 20, 7)), ("cube", 3, (3, 5, 7))])
def test_truncated_sort(zd, oracle_mod, monkeypatch, dist, dim, shift):
    """Builds of >= 2^20 points sort with 5 radix passes (key bits 24..63) and rank each
    run of equal 40-bit prefixes by (key, id); a run longer than 64 (here: every point
    in a 2^8-cube, so all prefixes are equal) redoes the sort with all 8 passes.  Either
    way the sorted arrays and the tree equal the full sort's and the oracle's."""
    n = (1 << 20) + 3
    if dist == "cube":
        pts = (zdgen.uniform(n, 3, seed=97) >> 13).astype(np.int32)   # [0, 2^8)^3
    else:
        pts = zdgen.points(dist, n, dim, seed=96)
    kw = {} if shift is None else dict(shift=shift)
    t = zd.zd_build(dev(pts), **kw)
    ex = t.zd_export()
    assert ex["info"]["sort_fallbacks"] == (1 if dist in ("cube", "dup") else 0)   # dup: an 8^3 grid
    monkeypatch.setenv("ZD_SORT_TRUNC", "0")
    u = zd.zd_build(dev(pts), **kw)
    ey = u.zd_export()
    assert ey["info"]["sort_fallbacks"] == 0
    assert np.array_equal(ex["keys"], ey["keys"]) and np.array_equal(ex["recs"], ey["recs"])
    assert np.array_equal(ex["leaf_start"], ey["leaf_start"]) and np.array_equal(ex["nodes"], ey["nodes"])
    if dist in ("uniform", "cube") and dim == 3 and shift is None:
        assert_same_structure(ex, oracle_mod.Tree(pts))
