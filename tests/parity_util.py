"""Helpers for GPU-vs-oracle parity: map the oracle's recursive tree onto the GPU's
flat in-order layout (leaf l = l-th leaf in key order; internal node i = the split
between leaf i and leaf i+1), so structure can be compared element by element."""
import numpy as np


def oracle_flat(t):
    """Oracle tree -> dict(leaf_start, leaf_parent, nodes[ni, words]) in the GPU layout."""
    nd = t.nodes()
    dim = t.dim
    split = nd["split"]
    leaves = np.nonzero(split < 0)[0]
    internal = np.nonzero(split >= 0)[0]
    leaves = leaves[np.argsort(nd["lo"][leaves], kind="stable")]
    # the split position of an internal node is where its right child starts
    pos = nd["lo"][nd["right"][internal]] if len(internal) else np.zeros(0, np.int64)
    internal = internal[np.argsort(pos, kind="stable")]
    ref = np.zeros(len(split), np.int64)
    ref[leaves] = ~np.arange(len(leaves))
    ref[internal] = np.arange(len(internal))
    leaf_start = np.concatenate([nd["lo"][leaves], [t.n]]).astype(np.int32)
    if t.n == 0:
        leaf_start = np.array([0, 0], np.int32)
    leaf_parent = np.where(nd["parent"][leaves] >= 0, ref[np.maximum(nd["parent"][leaves], 0)], -1).astype(np.int32)
    words = 4 * dim + 4
    nodes = np.zeros((len(internal), words), np.int32)
    for i, v in enumerate(internal):
        L, R = nd["left"][v], nd["right"][v]
        nodes[i, 0:dim] = nd["bmin"][L][:dim]
        nodes[i, dim:2 * dim] = nd["bmax"][L][:dim]
        nodes[i, 2 * dim:3 * dim] = nd["bmin"][R][:dim]
        nodes[i, 3 * dim:4 * dim] = nd["bmax"][R][:dim]
        nodes[i, 4 * dim] = ref[L]
        nodes[i, 4 * dim + 1] = ref[R]
        nodes[i, 4 * dim + 2] = ref[nd["parent"][v]] if nd["parent"][v] >= 0 else -1
        nodes[i, 4 * dim + 3] = split[v]
    root = ref[nd["root"]]
    return dict(leaf_start=leaf_start, leaf_parent=leaf_parent, nodes=nodes, root=int(root))


def assert_same_structure(gpu_export, t):
    exp = oracle_flat(t)
    keys, ids, coords = t.sorted_points()
    g = gpu_export
    assert np.array_equal(g["keys"], keys), "sorted keys differ"
    assert np.array_equal(g["recs"][:, 3], ids), "sorted ids differ"
    assert np.array_equal(g["recs"][:, :t.dim], coords[:, :t.dim]), "decoded coordinates differ"
    assert np.array_equal(g["leaf_start"], exp["leaf_start"]), "leaf boundaries differ"
    assert np.array_equal(g["leaf_parent"], exp["leaf_parent"]), "leaf parents differ"
    assert np.array_equal(g["nodes"], exp["nodes"]), "internal nodes differ"
    assert g["info"]["root"] == exp["root"]
    assert g["info"]["n_internal"] == len(exp["nodes"])


def first_row_mismatch(a_idx, a_d, b_idx, b_d):
    bad = np.nonzero(np.any(a_idx != b_idx, axis=1) | np.any(a_d != b_d, axis=1))[0]
    return bad
