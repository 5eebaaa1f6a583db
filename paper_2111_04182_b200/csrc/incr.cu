// incr.cu — NEXT-2 (part): insert fast path for batches that keep the canonical
// topology (Fig. 4; Alg. 4 P:354-381 read
// canonically, reading R17).
//
// A batch leaves the canonical tree's topology unchanged when every new key lies in
// the Morton cell of the leaf its bits route it to (it shares all key bits at and
// above the parent's split bit with that leaf's keys) and no leaf grows past the leaf
// size.  Then every node keeps its split bit (the highest differing bit of its keys
// cannot change: the new key differs from the leaf's keys only below the parent's
// split bit), no leaf splits and no internal node collapses — the tree of the new
// multiset has the same nodes, only with more points.  What changes:
//   * sorted keys/records: the merge (update.cu), as for any insert;
//   * point positions: leaf_start[l] += (inserted keys in leaves < l), pt_leaf, each
//     node's mid, its leaf-child point ranges and pos_range;
//   * boxes: each new point widens the child boxes on its leaf-to-root path
//     (min/max, so atomics give the exact tight boxes).
// Anything else (a key outside its leaf's cell, an overflowing leaf, an empty tree)
// takes the full canonical rebuild.
#include <climits>

#include "common.cuh"
#include "internal.h"

namespace zd {
namespace {

// Bit-located leaf of each (sorted) batch key + the cell check.
template <int DIM>
__global__ void __launch_bounds__(256) incr_locate_kernel(const uint64_t* __restrict__ bkeys, int32_t m,
                                                          const Node<DIM>* __restrict__ nodes,
                                                          const int32_t* __restrict__ split_bit,
                                                          const int32_t* __restrict__ meta,
                                                          const int32_t* __restrict__ leaf_start,
                                                          const uint64_t* __restrict__ keys, int32_t* __restrict__ bleaf,
                                                          int* __restrict__ bad) {
    const int32_t i = blockIdx.x * 256 + threadIdx.x;
    if (i >= m) return;
    const uint64_t key = __ldg(bkeys + i);
    int32_t cur = __ldg(meta + 1);
    if (cur < 0) { atomicOr(bad, 1); return; }   // single-leaf tree: full rebuild
    int32_t leaf = 0, pb = 0;
    while (true) {
        pb = __ldg(split_bit + cur);
        const bool right = (key >> pb) & 1u;
        const int32_t child = right ? __ldg(&nodes[cur].right) : __ldg(&nodes[cur].left);
        if (child < 0) { leaf = right ? cur + 1 : cur; break; }   // leaf children of node i: i, i+1
        cur = child;
    }
    const uint64_t k0 = __ldg(keys + __ldg(leaf_start + leaf));
    if (((key ^ k0) >> pb) != 0) atomicOr(bad, 1);   // outside the leaf's cell
    bleaf[i] = leaf;
}

// number of batch keys in leaves < l (bleaf is non-decreasing: sorted keys, checked cells)
__device__ __forceinline__ int32_t ins_before(const int32_t* __restrict__ bleaf, int32_t m, int32_t l) {
    int32_t lo = 0, hi = m;
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (__ldg(bleaf + mid) < l) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Leaf sizes after the insert must stay <= leaf_max (also checks monotone bleaf).
__global__ void __launch_bounds__(256) incr_check_kernel(const int32_t* __restrict__ bleaf, int32_t m,
                                                         const int32_t* __restrict__ leaf_start, int leaf_max,
                                                         int* __restrict__ bad) {
    const int32_t i = blockIdx.x * 256 + threadIdx.x;
    if (i >= m) return;
    const int32_t l = __ldg(bleaf + i);
    if (i > 0 && __ldg(bleaf + i - 1) > l) { atomicOr(bad, 1); return; }
    if (i == 0 || __ldg(bleaf + i - 1) != l) {   // first batch key of leaf l counts the leaf
        const int32_t c = ins_before(bleaf, m, l + 1) - i;
        if (__ldg(leaf_start + l + 1) - __ldg(leaf_start + l) + c > leaf_max) atomicOr(bad, 1);
    }
}

// leaf_start[l] += inserted keys before leaf l, l = 0 .. nleaves (in place)
__global__ void __launch_bounds__(256) incr_leaf_start_kernel(int32_t* __restrict__ leaf_start, int32_t nleaves,
                                                              const int32_t* __restrict__ bleaf, int32_t m) {
    const int32_t l = blockIdx.x * 256 + threadIdx.x;
    if (l > nleaves) return;
    leaf_start[l] += (l == nleaves) ? m : ins_before(bleaf, m, l);
}

// pt_leaf of every (new) sorted position, one thread per leaf
__global__ void __launch_bounds__(256) incr_pt_leaf_kernel(const int32_t* __restrict__ leaf_start, int32_t nleaves,
                                                           int32_t* __restrict__ pt_leaf) {
    const int32_t l = blockIdx.x * 256 + threadIdx.x;
    if (l >= nleaves) return;
    const int32_t e = __ldg(leaf_start + l + 1);
    for (int32_t p = __ldg(leaf_start + l); p < e; ++p) pt_leaf[p] = l;
}

// node position fields from the new leaf_start
template <int DIM>
__global__ void __launch_bounds__(256) incr_nodes_kernel(Node<DIM>* __restrict__ nodes, int32_t nb,
                                                         const int32_t* __restrict__ leaf_start,
                                                         const int32_t* __restrict__ range, int2* __restrict__ pos_range) {
    const int32_t i = blockIdx.x * 256 + threadIdx.x;
    if (i >= nb) return;
    Node<DIM>& nd = nodes[i];
    nd.mid = __ldg(leaf_start + i + 1);
    if (nd.left < 0) nd.left = ~__ldg(leaf_start + i);          // left leaf child = leaf i: ~start
    if (nd.right < 0) nd.right = ~__ldg(leaf_start + i + 2);    // right leaf child = leaf i+1: ~end
    pos_range[i] = make_int2(__ldg(leaf_start + __ldg(range + 2 * i)), __ldg(leaf_start + __ldg(range + 2 * i + 1) + 1));
}

// widen the child boxes on each new point's leaf-to-root path; box coordinates are
// non-negative (fp32 in 3D: ordered like their bit patterns; int32 in 2D)
template <int DIM>
__device__ __forceinline__ void widen(typename BoxT<DIM>::T* box, const int c[3]) {
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        if constexpr (DIM == 3) {
            const int v = __float_as_int((float)c[a]);
            atomicMin(reinterpret_cast<int*>(box + a), v);
            atomicMax(reinterpret_cast<int*>(box + DIM + a), v);
        } else {
            atomicMin(reinterpret_cast<int*>(box + a), c[a]);
            atomicMax(reinterpret_cast<int*>(box + DIM + a), c[a]);
        }
    }
}
template <int DIM>
__global__ void __launch_bounds__(256) incr_refit_kernel(Node<DIM>* __restrict__ nodes,
                                                         const int32_t* __restrict__ leaf_parent,
                                                         const int32_t* __restrict__ bleaf, const int4* __restrict__ brecs,
                                                         int32_t m) {
    const int32_t i = blockIdx.x * 256 + threadIdx.x;
    if (i >= m) return;
    const int4 r = __ldg(brecs + i);
    const int c[3] = {r.x, r.y, r.z};
    const int32_t l = __ldg(bleaf + i);
    int32_t P = __ldg(leaf_parent + l), C = -1;
    bool left = P == l;   // leaf l is the left child of node l
    while (P >= 0) {
        typename BoxT<DIM>::T* box = left ? nodes[P].lbox : nodes[P].rbox;
        // boxes only grow here, so a (possibly stale) box that already contains the
        // point proves every ancestor box will too (each widening of a child box is
        // followed by its own climb): stop
        bool inside = true;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            const typename BoxT<DIM>::T lo = __ldcg(box + a), hi = __ldcg(box + DIM + a);
            if constexpr (DIM == 3) {
                const float v = (float)c[a];   // exact: 21-bit coordinates
                inside = inside && lo <= v && v <= hi;
            } else {
                inside = inside && lo <= c[a] && c[a] <= hi;   // exact int32 (2D)
            }
        }
        if (inside) break;
        widen<DIM>(box, c);
        C = P;
        P = nodes[C].parent;
        if (P >= 0) left = nodes[P].left == C;
    }
}

}  // namespace

void incr_locate(int dim, const uint64_t* bkeys, int64_t m, const KnnArgs& t, const uint64_t* keys, int leaf_max,
                 int32_t* bleaf, int* bad, cudaStream_t st) {
    if (m <= 0) return;
    const unsigned grid = (unsigned)((m + 255) / 256);
    count_launch(2);
    if (dim == 2)
        incr_locate_kernel<2><<<grid, 256, 0, st>>>(bkeys, (int32_t)m, (const Node<2>*)t.nodes, t.split_bit, t.d_meta,
                                                    t.leaf_start, keys, bleaf, bad);
    else
        incr_locate_kernel<3><<<grid, 256, 0, st>>>(bkeys, (int32_t)m, (const Node<3>*)t.nodes, t.split_bit, t.d_meta,
                                                    t.leaf_start, keys, bleaf, bad);
    incr_check_kernel<<<grid, 256, 0, st>>>(bleaf, (int32_t)m, t.leaf_start, leaf_max, bad);
}

void incr_apply(int dim, int64_t nb, const int32_t* bleaf, const int4* brecs, int64_t m, int32_t* leaf_start,
                int32_t* pt_leaf, void* nodes, const int32_t* range, int2* pos_range, const int32_t* leaf_parent,
                cudaStream_t st) {
    const int32_t nleaves = (int32_t)nb + 1;
    count_launch(4);
    incr_leaf_start_kernel<<<(nleaves + 1 + 255) / 256, 256, 0, st>>>(leaf_start, nleaves, bleaf, (int32_t)m);
    incr_pt_leaf_kernel<<<(nleaves + 255) / 256, 256, 0, st>>>(leaf_start, nleaves, pt_leaf);
    const unsigned gn = (unsigned)std::max<int64_t>(1, (nb + 255) / 256);
    const unsigned gm = (unsigned)((m + 255) / 256);
    if (dim == 2) {
        incr_nodes_kernel<2><<<gn, 256, 0, st>>>((Node<2>*)nodes, (int32_t)nb, leaf_start, range, pos_range);
        incr_refit_kernel<2><<<gm, 256, 0, st>>>((Node<2>*)nodes, leaf_parent, bleaf, brecs, (int32_t)m);
    } else {
        incr_nodes_kernel<3><<<gn, 256, 0, st>>>((Node<3>*)nodes, (int32_t)nb, leaf_start, range, pos_range);
        incr_refit_kernel<3><<<gm, 256, 0, st>>>((Node<3>*)nodes, leaf_parent, bleaf, brecs, (int32_t)m);
    }
}

}  // namespace zd
