// common.cuh — shared device definitions of the zd-tree CUDA path (sm_100a).
// Product code only: nothing here is shared with oracle/ (the oracle has its own
// scalar bit-loop keys and recursive tree).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// Device-side bounds assertions for the debug build (-DZD_DEBUG; tests load it via
// ZD_LIB=<path>): the substitute for compute-sanitizer, which is unavailable here.
#ifdef ZD_DEBUG
#include <cassert>
#define ZD_DCHECK(c) assert(c)
#else
#define ZD_DCHECK(c) \
    do {             \
    } while (0)
#endif

namespace zd {

constexpr int kWarp = 32;
constexpr int kMaxLeaf = 32;      // ZD_LEAF_MAX_MAX
constexpr int kMaxDepth = 64;     // a path consumes a strictly lower key bit per level

template <int DIM> struct Dim;
template <> struct Dim<2> { static constexpr int B = 30; };   // 60-bit keys
template <> struct Dim<3> { static constexpr int B = 21; };   // 63-bit keys

// ---- Morton interleave (§1.1; dimension 0 most significant) ----
// Magic-number bit spreading: each coordinate's bits move to every DIM-th key bit.
__device__ __forceinline__ uint64_t spread2(uint32_t x) {
    uint64_t v = x & 0x7fffffffu;   // 30-bit coordinates, 31 with a random shift
    v = (v | (v << 16)) & 0x0000ffff0000ffffull;
    v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
    v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
    v = (v | (v << 2)) & 0x3333333333333333ull;
    v = (v | (v << 1)) & 0x5555555555555555ull;
    return v;
}
__device__ __forceinline__ uint32_t compact2(uint64_t v) {
    v &= 0x5555555555555555ull;
    v = (v ^ (v >> 1)) & 0x3333333333333333ull;
    v = (v ^ (v >> 2)) & 0x0f0f0f0f0f0f0f0full;
    v = (v ^ (v >> 4)) & 0x00ff00ff00ff00ffull;
    v = (v ^ (v >> 8)) & 0x0000ffff0000ffffull;
    v = (v ^ (v >> 16)) & 0x00000000ffffffffull;
    return (uint32_t)v;
}
__device__ __forceinline__ uint64_t spread3(uint32_t x) {
    uint64_t v = x & 0x1fffffu;
    v = (v | (v << 32)) & 0x001f00000000ffffull;
    v = (v | (v << 16)) & 0x001f0000ff0000ffull;
    v = (v | (v << 8)) & 0x100f00f00f00f00full;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}
__device__ __forceinline__ uint32_t compact3(uint64_t v) {
    v &= 0x1249249249249249ull;
    v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ull;
    v = (v ^ (v >> 4)) & 0x100f00f00f00f00full;
    v = (v ^ (v >> 8)) & 0x001f0000ff0000ffull;
    v = (v ^ (v >> 16)) & 0x001f00000000ffffull;
    v = (v ^ (v >> 32)) & 0x00000000001fffffull;
    return (uint32_t)v;
}

template <int DIM> __device__ __forceinline__ uint64_t morton(int x, int y, int z);
template <> __device__ __forceinline__ uint64_t morton<2>(int x, int y, int) {
    return (spread2((uint32_t)x) << 1) | spread2((uint32_t)y);
}
template <> __device__ __forceinline__ uint64_t morton<3>(int x, int y, int z) {
    return (spread3((uint32_t)x) << 2) | (spread3((uint32_t)y) << 1) | spread3((uint32_t)z);
}

// Record of a sorted point: coordinates decoded from the key (the interleave is a
// bijection on the 60/63 key bits) and the point id.
template <int DIM> __device__ __forceinline__ int4 decode_rec(uint64_t key, int id);
template <> __device__ __forceinline__ int4 decode_rec<2>(uint64_t key, int id) {
    return make_int4((int)compact2(key >> 1), (int)compact2(key), 0, id);
}
template <> __device__ __forceinline__ int4 decode_rec<3>(uint64_t key, int id) {
    return make_int4((int)compact3(key >> 2), (int)compact3(key >> 1), (int)compact3(key), id);
}

template <int DIM> __device__ __forceinline__ bool in_universe(int x, int y, int z) {
    constexpr uint32_t lim = 1u << Dim<DIM>::B;
    bool ok = (uint32_t)x < lim && (uint32_t)y < lim;
    if (DIM == 3) ok = ok && (uint32_t)z < lim;
    return ok;
}

// ---- tree layout ------------------------------------------------------------
// Internal node i (in-order: between leaf i and leaf i+1).  Both children's tight
// bounding boxes live in the parent so one 48/64-byte load decides the visit
// order and pruning of both children (Alg. 2's withinBox + nearer-child rule).
// Child refs: >= 0 an internal node; < 0 a leaf, encoded by its sorted point range
// so a leaf scan needs no further lookup:
//   left  leaf (= leaf i)   : left  = ~start, points [start, mid)
//   right leaf (= leaf i+1) : right = ~end,   points [mid, end)
// mid = first sorted position of the right subtree (= leaf_start[i+1]).  The split
// bit lives in a separate array (TreeBufs::split_bit); zd_export converts to the
// documented leaf-index form.
// Box coordinates: int32 in 2D (30-bit grid); fp32 in 3D, where every 21-bit grid
// coordinate is exact and the query's fp32 box tests have a proven error bound.
template <int DIM> struct BoxT { using T = int32_t; };
template <> struct BoxT<3> { using T = float; };
template <int DIM> struct alignas(16) Node {
    typename BoxT<DIM>::T lbox[2 * DIM];   // lo[DIM], hi[DIM]
    typename BoxT<DIM>::T rbox[2 * DIM];
    int32_t left, right, parent, mid;
};
static_assert(sizeof(Node<2>) == 48, "Node<2> layout");
static_assert(sizeof(Node<3>) == 64, "Node<3> layout");

__device__ __forceinline__ bool is_leaf_ref(int32_t r) { return r < 0; }

// block-wide exclusive scan of one uint32 per thread (blockDim.x == NT, NT % 32 == 0)
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t t = lane < NT / 32 ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < NT / 32) s_warp[lane] = t;   // inclusive warp totals
    }
    __syncthreads();
    uint32_t base = w > 0 ? s_warp[w - 1] : 0u;
    if (total) *total = s_warp[NT / 32 - 1];
    uint32_t r = base + x - v;
    __syncthreads();   // s_warp reusable after return
    return r;
}

// exclusive scan of block counts in place; block_cnt[nb] = total
static __global__ void __launch_bounds__(1024) scan_blocks_kernel(uint32_t* __restrict__ block_cnt, uint32_t nblocks) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < nblocks; b0 += 1024) {
        uint32_t i = b0 + threadIdx.x;
        uint32_t v = i < nblocks ? block_cnt[i] : 0u;
        uint32_t tot;
        uint32_t e = block_exclusive_scan<1024>(v, s_warp, &tot);
        uint32_t carry = s_carry;
        if (i < nblocks) block_cnt[i] = carry + e;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) block_cnt[nblocks] = s_carry;
}

}  // namespace zd
