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
    if (cur < 0) {   // single-leaf tree: full rebuild (bleaf stays a valid leaf index)
        bleaf[i] = 0;
        atomicOr(bad, 1);
        return;
    }
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
    if (i >= m || *(volatile int*)bad) return;   // refused already: leaf indices need not be valid
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

// ---- delete fast path ------------------------------------------------------------
// A delete batch keeps the canonical topology when no leaf is emptied and every
// internal node keeps more than leaf_max points: then both children of every node stay
// non-empty, so each node keeps its split bit (keys on both sides of it remain) and no
// node collapses into a leaf.  Positions shift down; boxes shrink, so they are
// recomputed along the paths of the leaves that lost points (a node is refit when its
// last dirty child arrives).

// per leaf: dead records (old positions, alive bitset by id), emptied-leaf check,
// block-exclusive scan into del_before, chunk totals into bsum.  The live leaf count
// comes from the device meta (meta[0] internal nodes, meta[1] root: a single-leaf tree
// takes the full rebuild), so the host needs no node count before the launch; a fixed
// grid walks the 256-leaf chunks (no blocks launched for the empty capacity).
__global__ void __launch_bounds__(256) decr_count_kernel(const int4* __restrict__ recs,
                                                         const int32_t* __restrict__ leaf_start,
                                                         const int32_t* __restrict__ meta,
                                                         const uint32_t* __restrict__ alive, int32_t* __restrict__ del_before,
                                                         uint32_t* __restrict__ bsum, int* __restrict__ bad) {
    __shared__ uint32_t s_warp[32];
    const int32_t nleaves = __ldg(meta) + 1;
    const int32_t nchunks = (nleaves + 255) / 256;
    if (blockIdx.x == 0 && threadIdx.x == 0 && __ldg(meta + 1) < 0) atomicOr(bad, 1);
    for (int32_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {   // block-uniform
        const int32_t l = ch * 256 + threadIdx.x;
        uint32_t c = 0;
        if (l < nleaves) {
            const int32_t s = __ldg(leaf_start + l), e = __ldg(leaf_start + l + 1);
            for (int32_t p = s; p < e; ++p) {
                const int32_t id = __ldg(recs + p).w;
                c += ((__ldg(alive + (id >> 5)) >> (id & 31)) & 1u) ? 0u : 1u;
            }
            if ((int32_t)c == e - s) atomicOr(bad, 1);   // leaf emptied
        }
        uint32_t total;
        const uint32_t ex = block_exclusive_scan<256>(c, s_warp, &total);
        if (l < nleaves) del_before[l] = (int32_t)ex;
        if (threadIdx.x == 0) bsum[ch] = total;
    }
}

// exclusive scan of the chunk totals (their count from the device meta); bsum[nchunks] = total
__global__ void __launch_bounds__(1024) decr_scan_kernel(uint32_t* __restrict__ bsum, const int32_t* __restrict__ meta) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    const uint32_t nchunks = (uint32_t)(__ldg(meta) + 1 + 255) / 256;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < nchunks; b0 += 1024) {
        const uint32_t i = b0 + threadIdx.x;
        const uint32_t v = i < nchunks ? bsum[i] : 0u;
        uint32_t tot;
        const uint32_t e = block_exclusive_scan<1024>(v, s_warp, &tot);
        const uint32_t carry = s_carry;
        if (i < nchunks) bsum[i] = carry + e;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) bsum[nchunks] = s_carry;
}

// del_before[l] += chunk offset; del_before[nleaves] = total
__global__ void __launch_bounds__(256) decr_fix_kernel(int32_t* __restrict__ del_before, const int32_t* __restrict__ meta,
                                                       const uint32_t* __restrict__ bsum) {
    const int32_t nleaves = __ldg(meta) + 1;
    const int32_t nchunks = (nleaves + 255) / 256;
    for (int32_t l = blockIdx.x * 256 + threadIdx.x; l <= nleaves; l += gridDim.x * 256) {
        if (l < nleaves) del_before[l] += (int32_t)__ldg(bsum + (l >> 8));
        else del_before[l] = (int32_t)__ldg(bsum + nchunks);
    }
}

// every internal node keeps > leaf_max points
__global__ void __launch_bounds__(256) decr_check_kernel(const int32_t* __restrict__ meta, const int32_t* __restrict__ range,
                                                         const int32_t* __restrict__ leaf_start,
                                                         const int32_t* __restrict__ del_before, int leaf_max,
                                                         int* __restrict__ bad) {
    const int32_t nb = __ldg(meta);
    for (int32_t i = blockIdx.x * 256 + threadIdx.x; i < nb; i += gridDim.x * 256) {
        const int32_t L = __ldg(range + 2 * i), R = __ldg(range + 2 * i + 1);
        const int32_t size = __ldg(leaf_start + R + 1) - __ldg(leaf_start + L);
        const int32_t del = __ldg(del_before + R + 1) - __ldg(del_before + L);
        if (size - del <= leaf_max) atomicOr(bad, 1);
    }
}

__global__ void __launch_bounds__(256) decr_leaf_start_kernel(int32_t* __restrict__ leaf_start, int32_t nleaves,
                                                              const int32_t* __restrict__ del_before) {
    const int32_t l = blockIdx.x * 256 + threadIdx.x;
    if (l <= nleaves) leaf_start[l] -= __ldg(del_before + l);
}

// mark, for each node, which children lie on a dirty leaf's path (bit 0 left, 1 right)
template <int DIM>
__global__ void __launch_bounds__(256) decr_mark_kernel(const Node<DIM>* __restrict__ nodes,
                                                        const int32_t* __restrict__ leaf_parent,
                                                        const int32_t* __restrict__ del_before, int32_t nleaves,
                                                        uint32_t* __restrict__ mark) {
    const int32_t l = blockIdx.x * 256 + threadIdx.x;
    if (l >= nleaves || __ldg(del_before + l + 1) == __ldg(del_before + l)) return;
    int32_t P = __ldg(leaf_parent + l), C = -1;
    uint32_t side = P == l ? 1u : 2u;   // leaf l is the left child of node l
    while (P >= 0) {
        if (atomicOr(mark + P, side) != 0u) break;   // the path above is marked already
        C = P;
        P = __ldg(&nodes[C].parent);
        if (P >= 0) side = __ldg(&nodes[P].left) == C ? 1u : 2u;
    }
}

template <int DIM>
__device__ __forceinline__ void put_box(typename BoxT<DIM>::T* dst, const typename BoxT<DIM>::T (&b)[2 * DIM]) {
#pragma unroll
    for (int a = 0; a < 2 * DIM; ++a) dst[a] = b[a];
}

// recompute dirty leaf boxes from the compacted records and refit up the marked paths
template <int DIM>
__global__ void __launch_bounds__(256) decr_refit_kernel(Node<DIM>* nodes, const int32_t* __restrict__ leaf_parent,
                                                         const int32_t* __restrict__ leaf_start_new,
                                                         const int32_t* __restrict__ del_before, int32_t nleaves,
                                                         const int4* __restrict__ recs, const uint32_t* __restrict__ mark,
                                                         uint32_t* arrived) {
    using T = typename BoxT<DIM>::T;
    const int32_t l = blockIdx.x * 256 + threadIdx.x;
    if (l >= nleaves || __ldg(del_before + l + 1) == __ldg(del_before + l)) return;
    int32_t lo[DIM], hi[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) { lo[a] = INT32_MAX; hi[a] = INT32_MIN; }
    const int32_t e = __ldg(leaf_start_new + l + 1);
    for (int32_t p = __ldg(leaf_start_new + l); p < e; ++p) {
        const int4 r = __ldg(recs + p);
        const int c[3] = {r.x, r.y, r.z};
#pragma unroll
        for (int a = 0; a < DIM; ++a) { lo[a] = min(lo[a], c[a]); hi[a] = max(hi[a], c[a]); }
    }
    T b[2 * DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) { b[a] = (T)lo[a]; b[DIM + a] = (T)hi[a]; }
    int32_t P = __ldg(leaf_parent + l), C = -1;
    bool left = P == l;
    while (P >= 0) {
        put_box<DIM>(left ? nodes[P].lbox : nodes[P].rbox, b);
        __threadfence();   // release: the box before the arrival
        const uint32_t need = __popc(__ldcg(mark + P));
        if (atomicAdd(arrived + P, 1u) + 1u < need) return;   // the other dirty child finishes P
        __threadfence();   // acquire: the sibling's box
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            const T l0 = __ldcg(nodes[P].lbox + a), r0 = __ldcg(nodes[P].rbox + a);
            const T l1 = __ldcg(nodes[P].lbox + DIM + a), r1 = __ldcg(nodes[P].rbox + DIM + a);
            b[a] = l0 < r0 ? l0 : r0;
            b[DIM + a] = l1 > r1 ? l1 : r1;
        }
        C = P;
        P = __ldcg(&nodes[C].parent);
        if (P >= 0) left = __ldcg(&nodes[P].left) == C;
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

namespace zd {

int decr_check(int64_t nb_cap, const int32_t* meta, const int4* recs_old, const int32_t* leaf_start,
               const uint32_t* alive, const int32_t* range, int leaf_max, int32_t* del_before, uint32_t* bsum, int* bad,
               cudaStream_t st) {
    // fixed grids over the device-side leaf / node counts (the capacity nb_cap may be
    // ~11x the node count: worst-case sized node buffers below 2^25 points)
    const int64_t nl_cap = nb_cap + 1;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * 8, (nl_cap + 255) / 256));
    count_launch(4);
    decr_count_kernel<<<g, 256, 0, st>>>(recs_old, leaf_start, meta, alive, del_before, bsum, bad);
    decr_scan_kernel<<<1, 1024, 0, st>>>(bsum, meta);
    decr_fix_kernel<<<g, 256, 0, st>>>(del_before, meta, bsum);
    if (nb_cap > 0) decr_check_kernel<<<g, 256, 0, st>>>(meta, range, leaf_start, del_before, leaf_max, bad);
    return 0;
}

void decr_apply(int dim, int64_t nb, const int32_t* del_before, int32_t* leaf_start, int32_t* pt_leaf, void* nodes,
                const int32_t* range, int2* pos_range, const int32_t* leaf_parent, const int4* recs_new, uint32_t* mark,
                uint32_t* arrived, cudaStream_t st) {
    const int32_t nleaves = (int32_t)nb + 1;
    const unsigned gl = (unsigned)((nleaves + 255) / 256), gn = (unsigned)std::max<int64_t>(1, (nb + 255) / 256);
    count_launch(5);
    decr_leaf_start_kernel<<<(nleaves + 1 + 255) / 256, 256, 0, st>>>(leaf_start, nleaves, del_before);
    incr_pt_leaf_kernel<<<gl, 256, 0, st>>>(leaf_start, nleaves, pt_leaf);
    if (dim == 2) {
        incr_nodes_kernel<2><<<gn, 256, 0, st>>>((Node<2>*)nodes, (int32_t)nb, leaf_start, range, pos_range);
        decr_mark_kernel<2><<<gl, 256, 0, st>>>((const Node<2>*)nodes, leaf_parent, del_before, nleaves, mark);
        decr_refit_kernel<2><<<gl, 256, 0, st>>>((Node<2>*)nodes, leaf_parent, leaf_start, del_before, nleaves, recs_new,
                                                 mark, arrived);
    } else {
        incr_nodes_kernel<3><<<gn, 256, 0, st>>>((Node<3>*)nodes, (int32_t)nb, leaf_start, range, pos_range);
        decr_mark_kernel<3><<<gl, 256, 0, st>>>((const Node<3>*)nodes, leaf_parent, del_before, nleaves, mark);
        decr_refit_kernel<3><<<gl, 256, 0, st>>>((Node<3>*)nodes, leaf_parent, leaf_start, del_before, nleaves, recs_new,
                                                 mark, arrived);
    }
}

}  // namespace zd
