// tree.cu — K4 canonical topology + K5 bottom-up bounding boxes.
//
// The tree is Alg. 1 buildTree with empty cuts skipped
// (P:463): node = sorted range [lo, hi); leaf iff hi-lo <= leaf_max or all keys
// equal; otherwise cut at b = msb(key[lo] ^ key[hi-1]) and split at the first index
// whose bit b is 1 (splitUsingBit).  Boxes are the tight per-axis bounds of a
// node's points ("two opposing corners"; SURVEY reading 7).
//
// Flat data-parallel construction (not the paper's fork-join recursion):
//  * delta_p = msb(key_p ^ key_{p+1}) for adjacent sorted keys (-1 if equal).  The
//    full radix tree is the Cartesian tree of delta: the node whose cut is at pair p
//    spans [L+1, R+1) where L / R are the nearest pairs left / right of p with a
//    larger delta.  That node holds more than leaf_max points and has distinct
//    keys ("big") iff delta_p >= 0 and R - L > leaf_max, which a thread decides by
//    looking at most leaf_max-1 pairs to each side (shared-memory window).
//  * Collapsing every small subtree into a leaf leaves exactly the big pairs as
//    internal nodes; the leaves are the gaps between consecutive big pairs, and the
//    internal nodes form the Cartesian tree of the big pairs' deltas (nearest larger
//    neighbours are ancestors, hence big).  A scan over the flags numbers internal
//    nodes in-order: internal node i separates leaf i from leaf i+1.
//  * One thread per leaf computes the leaf box and climbs: the parent of a node
//    spanning leaves [Ll, Rl] is the boundary pair with the smaller delta (the two
//    boundary deltas always differ).  The first child to arrive at a parent stops;
//    the second merges both boxes and continues (atomic arrival counter).  Linear
//    work, one pass, no recursion.
#include <algorithm>
#include <cuda/atomic>

#include "common.cuh"
#include "internal.h"

namespace zd {

namespace {

constexpr int TT = 256;
#ifndef ZD_TPI
#define ZD_TPI 4
#endif
constexpr int TPI = ZD_TPI;   // pairs per thread in the flags / compact kernels
constexpr int TTILE = TT * TPI;   // pairs per block
constexpr int HALO = kMaxLeaf;

__device__ __forceinline__ int delta_of(uint64_t a, uint64_t b) {
    uint64_t x = a ^ b;
    return x ? 63 - __clzll((long long)x) : -1;
}

// 16-bit mask of the bytes s[p .. p+15] that are > d, from word loads of shared
// memory and funnel shifts.  Bytes hold delta + 1 in [0, 63] or 128 (range boundary)
// and 1 <= d <= 63, so adding 127 - d to every byte never carries into the next one
// and sets a byte's top bit exactly when the byte is > d: one 32-bit add per 4 bytes.
__device__ __forceinline__ uint32_t greater_mask16(const uint8_t* s, int p, int d) {
    const int a = p & ~3, sh = (p & 3) * 8;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(s + a);
    uint32_t words[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) words[i] = w[i];
    const uint32_t bias = (uint32_t)(127 - d) * 0x01010101u;
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t v = __funnelshift_r(words[i], words[i + 1], sh);
        const uint32_t g = (v + bias) & 0x80808080u;               // 0x80 in each greater byte
        m |= ((g * 0x00204081u) >> 28) << (4 * i);                 // byte top bits -> 4 bits
    }
    return m;
}

__global__ void __launch_bounds__(TT) flags_kernel(const uint64_t* __restrict__ keys, uint32_t n, int leaf_max,
                                                   uint8_t* __restrict__ flags, uint32_t* __restrict__ block_cnt) {
    __shared__ __align__(16) uint8_t s_delta[TTILE + 2 * HALO + 8];   // delta + 1; 128 = boundary
    __shared__ uint32_t s_warp[32];
    const int64_t base = (int64_t)blockIdx.x * TTILE;
    const int64_t npairs = (int64_t)n - 1;
    for (int t = threadIdx.x; t < TTILE + 2 * HALO; t += TT) {
        int64_t p = base - HALO + t;
        // out-of-range pairs act as +infinity: the range boundary
        s_delta[t] = (p >= 0 && p < npairs) ? (uint8_t)(delta_of(keys[p], keys[p + 1]) + 1) : (uint8_t)128;
    }
    __syncthreads();
    const int W = leaf_max - 1;
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < TPI; ++i) {
        const int off = threadIdx.x + i * TT;
        const int64_t p = base + off;
        if (p >= npairs) continue;
        const int c = HALO + off;
        const int d = s_delta[c];   // delta + 1
        bool big = false;
        if (d >= 1) {
            int l = 1, r = 1;
            if (W <= 15) {
                // branch-free: nearest larger delta within 16 bytes on each side via
                // SIMD byte compares (bit k of gl: byte c-16+k > d; of gr: byte c+1+k > d)
                const uint32_t gl = greater_mask16(s_delta, c - 16, d);
                const uint32_t gr = greater_mask16(s_delta, c + 1, d);
                const uint32_t ml = gl & (0xffffu << (16 - W));   // positions c-W .. c-1
                const uint32_t mr = gr & ((1u << W) - 1u);         // positions c+1 .. c+W
                l = ml ? 16 - (31 - __clz(ml)) : W + 1;
                r = mr ? __ffs(mr) : W + 1;
            } else {
                while (l <= W && s_delta[c - l] <= d) ++l;
                while (r <= W && s_delta[c + r] <= d) ++r;
            }
            big = (l + r) > leaf_max;   // node size = l + r
        }
        flags[p] = big;
        cnt += big;
    }
    uint32_t total;
    block_exclusive_scan<TT>(cnt, s_warp, &total);
    if (threadIdx.x == 0) block_cnt[blockIdx.x] = total;
}

__global__ void __launch_bounds__(TT) compact_kernel(const uint8_t* __restrict__ flags, const uint64_t* __restrict__ keys,
                                                     uint32_t n, const uint32_t* __restrict__ block_off,
                                                     int32_t* __restrict__ split_bit, int32_t* __restrict__ leaf_start,
                                                     int32_t* __restrict__ pt_leaf, int32_t* __restrict__ meta,
                                                     uint32_t* __restrict__ visit, int32_t* __restrict__ node_words,
                                                     int nw) {
    __shared__ uint32_t s_warp[32];
    const int64_t base = (int64_t)blockIdx.x * TTILE + threadIdx.x * TPI;   // blocked per thread
    const int64_t npairs = (int64_t)n - 1;
    uint8_t f[TPI];
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < TPI; ++i) {
        int64_t p = base + i;
        f[i] = p < npairs ? flags[p] : 0;
        c += f[i];
    }
    uint32_t run = block_off[blockIdx.x] + block_exclusive_scan<TT>(c, s_warp, nullptr);
#pragma unroll
    for (int i = 0; i < TPI; ++i) {
        int64_t p = base + i;
        if (p < n) pt_leaf[p] = (int32_t)run;   // leaf = number of big pairs before p
        if (f[i]) {
            split_bit[run] = delta_of(keys[p], keys[p + 1]);
            leaf_start[run + 1] = (int32_t)(p + 1);
            node_words[(size_t)run * nw + nw - 1] = (int32_t)(p + 1);   // Node::mid
            visit[run] = 0u;   // bottom-up arrival counter of internal node `run`
            ++run;
        }
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        uint32_t nb = block_off[gridDim.x];
        meta[0] = (int32_t)nb;
        meta[1] = nb == 0 ? ~0 : -1;   // root: single leaf, or set by the bottom-up pass
        leaf_start[0] = 0;
        leaf_start[nb + 1] = (int32_t)n;
    }
}

// K4 in one pass (builds with node buffers sized for the worst case): the flags of
// flags_kernel, the internal-node numbering of compact_kernel, with the tile's global
// offset resolved by a decoupled look-back over the preceding tiles instead of a
// separate block scan and a second read of the keys.  Tiles are taken in launch order
// from a counter (every predecessor of a tile is resident or done).  Status words:
// bits 31:30 = 1 aggregate / 2 inclusive prefix, bits 29:0 = the count (nb < n < 2^30).
constexpr uint32_t kTopoVal = (1u << 30) - 1, kTopoAgg = 1u << 30, kTopoInc = 2u << 30;
#ifndef ZD_TOPO_TPI
#define ZD_TOPO_TPI 8
#endif
constexpr int TPI2 = ZD_TOPO_TPI;      // pairs per thread in topo_kernel
constexpr int TTILE2 = TT * TPI2;      // pairs per topo_kernel tile
static_assert(TPI2 % 4 == 0, "topo_kernel stores a thread's pt_leaf entries as int4s");

__global__ void __launch_bounds__(TT) topo_kernel(const uint64_t* __restrict__ keys, uint32_t n, int leaf_max,
                                                  uint32_t* status, uint32_t ntiles, int32_t* __restrict__ split_bit,
                                                  int32_t* __restrict__ leaf_start, int32_t* __restrict__ pt_leaf,
                                                  int32_t* __restrict__ meta, uint32_t* __restrict__ visit,
                                                  int32_t* __restrict__ node_words, int nw) {
    __shared__ __align__(16) uint8_t s_delta[TTILE2 + 2 * HALO + 8];   // delta + 1; 128 = boundary
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_tile, s_excl;
    uint32_t* counter = status + ntiles;
    if (threadIdx.x == 0) {
        const uint32_t t = atomicAdd(counter, 1u);
        s_tile = t;
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t base = (int64_t)tile * TTILE2;
    const int64_t npairs = (int64_t)n - 1;
    for (int t = threadIdx.x; t < TTILE2 + 2 * HALO; t += TT) {
        const int64_t p = base - HALO + t;
        s_delta[t] = (p >= 0 && p < npairs) ? (uint8_t)(delta_of(keys[p], keys[p + 1]) + 1) : (uint8_t)128;
    }
    __syncthreads();
    const int W = leaf_max - 1;
    uint8_t f[TPI2];
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < TPI2; ++i) {
        const int off = threadIdx.x * TPI2 + i;   // blocked: a thread's pairs are consecutive
        const int64_t p = base + off;
        const int c = HALO + off;
        const int d = s_delta[c];   // delta + 1
        bool big = false;
        if (p < npairs && d >= 1) {
            int l = 1, r = 1;
            if (W <= 15) {
                const uint32_t gl = greater_mask16(s_delta, c - 16, d);
                const uint32_t gr = greater_mask16(s_delta, c + 1, d);
                const uint32_t ml = gl & (0xffffu << (16 - W));
                const uint32_t mr = gr & ((1u << W) - 1u);
                l = ml ? 16 - (31 - __clz(ml)) : W + 1;
                r = mr ? __ffs(mr) : W + 1;
            } else {
                while (l <= W && s_delta[c - l] <= d) ++l;
                while (r <= W && s_delta[c + r] <= d) ++r;
            }
            big = (l + r) > leaf_max;
        }
        f[i] = big;
        cnt += big;
    }
    uint32_t total;
    const uint32_t local = block_exclusive_scan<TT>(cnt, s_warp, &total);
    // decoupled look-back: one warp folds the predecessors' words 32 at a time
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        uint32_t* mine = status + tile;
        if (lane == 0) {
            cuda::atomic_ref<uint32_t, cuda::thread_scope_device>(*mine).store(
                (tile == 0 ? kTopoInc : kTopoAgg) | total, cuda::memory_order_relaxed);
        }
        uint32_t excl = 0;
        int64_t t = (int64_t)tile - 1;
        while (t >= 0) {
            const int64_t q = t - lane;
            uint32_t v = kTopoInc;   // past tile 0: an inclusive zero
            if (q >= 0) {
                do {
                    v = cuda::atomic_ref<uint32_t, cuda::thread_scope_device>(status[q]).load(cuda::memory_order_relaxed);
                } while ((v & ~kTopoVal) == 0);
            }
            const uint32_t inc = __ballot_sync(0xffffffffu, (v & ~kTopoVal) == kTopoInc);
            const int stop = inc ? __ffs(inc) - 1 : 31;   // nearest inclusive predecessor in the window
            uint32_t x = lane <= stop ? (v & kTopoVal) : 0u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            excl += x;
            if (inc) break;
            t -= 32;
        }
        if (lane == 0) {
            if (tile > 0)
                cuda::atomic_ref<uint32_t, cuda::thread_scope_device>(*mine).store(kTopoInc | (excl + total),
                                                                                   cuda::memory_order_relaxed);
            s_excl = excl;
            if (tile == ntiles - 1) {
                const uint32_t nb = excl + total;
                meta[0] = (int32_t)nb;
                meta[1] = nb == 0 ? ~0 : -1;   // root: single leaf, or set by the bottom-up pass
                leaf_start[0] = 0;
                leaf_start[nb + 1] = (int32_t)n;
                *counter = 0;                  // every tile id is taken: reset for the next build
            }
        }
    }
    __syncthreads();
    uint32_t run = s_excl + local;
    const int64_t p0 = base + threadIdx.x * TPI2;
    int32_t pl[TPI2];
#pragma unroll
    for (int i = 0; i < TPI2; ++i) {
        const int64_t p = p0 + i;
        pl[i] = (int32_t)run;   // leaf = number of big pairs before p
        if (f[i]) {
            split_bit[run] = s_delta[HALO + threadIdx.x * TPI2 + i] - 1;
            leaf_start[run + 1] = (int32_t)(p + 1);
            node_words[(size_t)run * nw + nw - 1] = (int32_t)(p + 1);   // Node::mid
            visit[run] = 0u;
            ++run;
        }
    }
    if (p0 + TPI2 <= (int64_t)n) {
#pragma unroll
        for (int i = 0; i < TPI2; i += 4)
            *reinterpret_cast<int4*>(pt_leaf + p0 + i) = make_int4(pl[i], pl[i + 1], pl[i + 2], pl[i + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < TPI2; ++i)
            if (p0 + i < (int64_t)n) pt_leaf[p0 + i] = pl[i];
    }
}

// a child box into its parent node: vector stores (3D: fp32 pairs at 8-byte offsets;
// 2D: one int4 at a 16-byte offset); the conversion is exact (3D: < 2^21)
template <int DIM>
__device__ __forceinline__ void store_box(typename BoxT<DIM>::T* dst, const int32_t (&b)[2 * DIM]) {
    if constexpr (DIM == 3) {
        float2* d = reinterpret_cast<float2*>(dst);
        d[0] = make_float2((float)b[0], (float)b[1]);
        d[1] = make_float2((float)b[2], (float)b[3]);
        d[2] = make_float2((float)b[4], (float)b[5]);
    } else {
        *reinterpret_cast<int4*>(dst) = make_int4(b[0], b[1], b[2], b[3]);
    }
}

// One block per window of BW consecutive leaves.  An internal node whose whole leaf
// range lies in the window ("local") gets both of its arrivals from this block: a node's
// range is bounded by the nearest larger split bit on each side (the canonical tree is
// the Cartesian tree of the split bits), found by prefix / suffix max scans of the
// window's split bits.
//   1. leaf boxes, then the climb through local nodes: children's boxes, leaf bounds,
//      refs and parent links go through shared memory only (block-scoped
//      release/acquire on a shared arrival counter; no global store or device fence
//      inside the dependent chain);
//   2. after a block barrier, thread t writes the complete record of local node b0+t
//      (one contiguous 48/64-byte store per thread), its leaf bounds and point range,
//      and leaf b0+t's parent;
//   3. the threads that reached a window-crossing parent continue with device-scope
//      acq_rel arrival counters in global memory (a crossing node's ancestors all cross).
#ifndef ZD_BU_WINDOW
#define ZD_BU_WINDOW 128
#endif
constexpr int BW = ZD_BU_WINDOW;   // leaves per bottom-up block (window)
#ifndef ZD_LEAF_UNROLL
#define ZD_LEAF_UNROLL 4
#endif
constexpr int kLeafUnroll = ZD_LEAF_UNROLL;   // leaf-box record loads in flight per thread

template <int DIM>
__global__ void __launch_bounds__(BW) bottom_up_kernel(const int4* __restrict__ recs, const int32_t* __restrict__ leaf_start,
                                                        const int32_t* __restrict__ split_bit, int32_t* meta,
                                                        Node<DIM>* nodes, int32_t* __restrict__ leaf_parent,
                                                        uint32_t* visit, int32_t* range, int2* __restrict__ pos_range) {
    using BT = typename BoxT<DIM>::T;
    __shared__ int32_t s_sb[BW + 1];      // split bits of nodes b0-1 .. b0+BW-1 (INT32_MAX outside [0, nb))
    __shared__ int32_t s_ls[BW + 1];      // leaf_start[b0 .. b0+BW]
    __shared__ uint8_t s_local[BW];       // node b0+t finishes inside this block
    __shared__ uint32_t s_visit[BW];      // block-local arrival counters
    __shared__ int32_t s_rng[BW][2];      // local nodes: children's leaf bounds (L of left, R of right)
    __shared__ int32_t s_cref[BW][2];     // local nodes: child refs
    __shared__ int32_t s_par[BW];         // local nodes: parent (-1 until a child of the parent sets it)
    __shared__ __align__(8) int32_t s_box[BW][2][2 * DIM];   // local nodes: children's boxes
    const int32_t nb = meta[0];
    const int32_t b0 = blockIdx.x * BW;
    if (b0 > nb) return;                  // block-uniform
    const int t = threadIdx.x;
    for (int i = t; i <= BW; i += BW) {
        const int32_t q = b0 - 1 + i;
        s_sb[i] = (q >= 0 && q < nb) ? __ldg(split_bit + q) : INT32_MAX;
        s_ls[i] = b0 + i <= nb + 1 ? leaf_start[b0 + i] : 0;
    }
    __syncthreads();
    {
        __shared__ int32_t s_wmax[2][BW / 32];
        __shared__ int32_t s_suf[BW];
        const int lane = t & 31, wi = t >> 5;
        int32_t pv = s_sb[t], sv = s_sb[t + 1];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, pv, o);
            const int32_t z = __shfl_down_sync(0xffffffffu, sv, o);
            if (lane >= o) pv = max(pv, y);
            if (lane + o < 32) sv = max(sv, z);
        }
        if (lane == 31) s_wmax[0][wi] = pv;
        if (lane == 0) s_wmax[1][wi] = sv;
        __syncthreads();
        for (int w = 0; w < wi; ++w) pv = max(pv, s_wmax[0][w]);              // max s_sb[0..t]
        for (int w = wi + 1; w < BW / 32; ++w) sv = max(sv, s_wmax[1][w]);     // max s_sb[t+1..BW]
        s_suf[t] = sv;
        __syncthreads();
        bool loc = false;
        if (b0 + t < nb) {
            const int32_t d = s_sb[t + 1];
            const int32_t rmax = t + 1 < BW ? s_suf[t + 1] : INT32_MIN;     // max s_sb[t+2..BW]
            loc = pv > d && rmax > d;
        }
        s_local[t] = loc;
        s_visit[t] = 0u;
        s_par[t] = -1;
    }
    __syncthreads();
    const int32_t l = b0 + t;
    if (nb == 0) {                        // block-uniform: a single leaf (only block 0 gets here)
        if (t == 0) leaf_parent[0] = -1;
        return;
    }
    auto sbit = [&](int32_t q) { return (q >= b0 - 1 && q < b0 + BW) ? s_sb[q - b0 + 1] : __ldg(split_bit + q); };
    auto lstart = [&](int32_t q) { return (q >= b0 && q <= b0 + BW) ? s_ls[q - b0] : __ldg(leaf_start + q); };
    // parent of the subtree spanning leaves [L, R]: the boundary node with the smaller split bit
    auto parent_of = [&](int32_t L, int32_t R, bool& as_right) {
        if (L == 0) { as_right = false; return R; }
        if (R == nb) { as_right = true; return L - 1; }
        if (sbit(L - 1) < sbit(R)) { as_right = true; return L - 1; }
        as_right = false;
        return R;
    };
    int32_t bb[2 * DIM];
    int32_t L = l, R = l, ref = -1, s = 0, e = 0, lp = -1;
    bool pending = false;
#pragma unroll
    for (int a = 0; a < DIM; ++a) { bb[a] = INT32_MAX; bb[DIM + a] = INT32_MIN; }
    if (l <= nb) {
        s = s_ls[t];
        e = lstart(l + 1);
        // leaf box from its records (independent loads, unrolled)
#pragma unroll kLeafUnroll
        for (int32_t j = s; j < e; ++j) {
            const int4 r = __ldg(recs + j);
            const int c[3] = {r.x, r.y, r.z};
#pragma unroll
            for (int a = 0; a < DIM; ++a) { bb[a] = min(bb[a], c[a]); bb[DIM + a] = max(bb[DIM + a], c[a]); }
        }
        // window-relative climb: the subtree's leaves stay inside the window, so both
        // boundary split bits are in s_sb (the INT32_MAX sentinels outside [0, nb) make
        // L == 0 choose R and R == nb choose L - 1, as parent_of does)
        int Lr = t, Rr = t;
        while (true) {
            const bool as_right = s_sb[Lr] < s_sb[Rr + 1];
            const int pi = as_right ? Lr - 1 : Rr;
            if (pi < 0 || pi >= BW || !s_local[pi]) { pending = true; break; }
            const int side = as_right ? 1 : 0;
            const int32_t par = b0 + pi;
#pragma unroll
            for (int a = 0; a < DIM; ++a)
                reinterpret_cast<int2*>(s_box[pi][side])[a] = make_int2(bb[2 * a], bb[2 * a + 1]);
            s_rng[pi][side] = b0 + (as_right ? Rr : Lr);
            // a leaf child is encoded by its point range: left = ~start, right = ~end
            s_cref[pi][side] = ref >= 0 ? ref : (as_right ? ~e : ~s);
            if (ref < 0) lp = par; else s_par[ref - b0] = par;   // a local node's children are local
            __threadfence_block();
            if (atomicAdd(&s_visit[pi], 1u) == 0) break;          // first child: the sibling finishes the parent
            __threadfence_block();
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                const int2 v = reinterpret_cast<const int2*>(s_box[pi][side ^ 1])[a];
                const int32_t o0 = v.x, o1 = v.y;   // entries 2a, 2a+1 of the sibling's box
                if (2 * a < DIM) bb[2 * a] = min(bb[2 * a], o0); else bb[2 * a] = max(bb[2 * a], o0);
                if (2 * a + 1 < DIM) bb[2 * a + 1] = min(bb[2 * a + 1], o1); else bb[2 * a + 1] = max(bb[2 * a + 1], o1);
            }
            if (as_right) Lr = s_rng[pi][0] - b0; else Rr = s_rng[pi][1] - b0;
            ref = par;
            if (b0 + Lr == 0 && b0 + Rr == nb) { meta[1] = par; break; }      // the root is local: its parent stays -1
        }
        L = b0 + Lr;
        R = b0 + Rr;
    }
    __syncthreads();
    if (lp >= 0) leaf_parent[l] = lp;
    if (l < nb && s_local[t]) {
        Node<DIM> nd;
#pragma unroll
        for (int a = 0; a < 2 * DIM; ++a) {
            nd.lbox[a] = (BT)s_box[t][0][a];   // exact (3D: < 2^21)
            nd.rbox[a] = (BT)s_box[t][1][a];
        }
        nd.left = s_cref[t][0];
        nd.right = s_cref[t][1];
        nd.parent = s_par[t];
        nd.mid = s_ls[t + 1];
        int4* dst = reinterpret_cast<int4*>(nodes + l);
        const int4* src = reinterpret_cast<const int4*>(&nd);
#pragma unroll
        for (int i = 0; i < (int)(sizeof(Node<DIM>) / 16); ++i) dst[i] = src[i];
        const int32_t nl = s_rng[t][0], nr = s_rng[t][1];
        *reinterpret_cast<int2*>(range + 2 * l) = make_int2(nl, nr);
        pos_range[l] = make_int2(s_ls[nl - b0], s_ls[nr + 1 - b0]);
    }
    __syncthreads();   // the records written above precede the parent links written below
    if (!pending) return;
    while (true) {
        bool as_right;
        const int32_t par = parent_of(L, R, as_right);
        ZD_DCHECK(par >= 0 && par < nb && L >= 0 && R <= nb);
        Node<DIM>* P = nodes + par;
        const int32_t cref = ref >= 0 ? ref : (as_right ? ~e : ~s);
        if (as_right) { store_box<DIM>(P->rbox, bb); P->right = cref; }
        else { store_box<DIM>(P->lbox, bb); P->left = cref; }
        range[2 * par + (as_right ? 1 : 0)] = as_right ? R : L;   // leaf bounds (also read by the delete check)
        if (ref < 0) leaf_parent[l] = par; else nodes[ref].parent = par;
        // release: our writes are visible before the count; acquire: the second arriver sees its sibling's
        const uint32_t arrived =
            cuda::atomic_ref<uint32_t, cuda::thread_scope_device>(visit[par]).fetch_add(1u, cuda::memory_order_acq_rel);
        if (arrived == 0) break;   // first child: the sibling finishes the parent
        const BT* sb = as_right ? P->lbox : P->rbox;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            bb[a] = min(bb[a], (int32_t)__ldcg(sb + a));
            bb[DIM + a] = max(bb[DIM + a], (int32_t)__ldcg(sb + DIM + a));
        }
        if (as_right) L = __ldcg(range + 2 * par); else R = __ldcg(range + 2 * par + 1);
        pos_range[par] = make_int2(lstart(L), lstart(R + 1));
        ref = par;
        if (L == 0 && R == nb) { P->parent = -1; meta[1] = par; break; }
    }
}

template <int DIM>
__global__ void __launch_bounds__(256) export_nodes_kernel(const Node<DIM>* __restrict__ nodes,
                                                           const int32_t* __restrict__ split_bit, int64_t nb,
                                                           int32_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (i >= nb) return;
    const Node<DIM> nd = nodes[i];
    int32_t* o = out + i * (4 * DIM + 4);
#pragma unroll
    for (int a = 0; a < 2 * DIM; ++a) { o[a] = (int32_t)nd.lbox[a]; o[2 * DIM + a] = (int32_t)nd.rbox[a]; }
    o[4 * DIM] = nd.left >= 0 ? nd.left : ~(int32_t)i;             // left leaf child = leaf i
    o[4 * DIM + 1] = nd.right >= 0 ? nd.right : ~(int32_t)(i + 1);  // right leaf child = leaf i+1
    o[4 * DIM + 2] = nd.parent;
    o[4 * DIM + 3] = split_bit[i];
}

}  // namespace

void export_nodes(int dim, const void* nodes, const int32_t* split_bit, int64_t nb, int32_t* out, cudaStream_t st) {
    if (nb <= 0) return;
    const unsigned grid = (unsigned)((nb + 255) / 256);
    count_launch(1);
    if (dim == 2) export_nodes_kernel<2><<<grid, 256, 0, st>>>((const Node<2>*)nodes, split_bit, nb, out);
    else export_nodes_kernel<3><<<grid, 256, 0, st>>>((const Node<3>*)nodes, split_bit, nb, out);
}

// blocks of the flags / compact kernels: they must cover every position (compact writes
// pt_leaf of positions 0 .. n-1) as well as every pair 0 .. n-2
size_t tree_blocks(int64_t n) { return (size_t)std::max<int64_t>(1, (n + TTILE - 1) / TTILE); }

void topology_flags(const uint64_t* keys, int64_t n, int leaf_max, const TreeBufs& t, cudaStream_t st) {
    const size_t nblk = tree_blocks(n);
    flags_kernel<<<nblk, TT, 0, st>>>(keys, (uint32_t)n, leaf_max, t.flags, t.block_cnt);
    scan_blocks_kernel<<<1, 1024, 0, st>>>(t.block_cnt, (uint32_t)nblk);
    count_launch(2);
}

static void topology_boxes(int dim, const int4* recs, int64_t n, const TreeBufs& t, cudaStream_t st);

void topology_finish(int dim, const uint64_t* keys, const int4* recs, int64_t n, const TreeBufs& t, cudaStream_t st,
                     cudaEvent_t ev_mid) {
    const int nw = dim == 2 ? (int)(sizeof(Node<2>) / 4) : (int)(sizeof(Node<3>) / 4);
    compact_kernel<<<tree_blocks(n), TT, 0, st>>>(t.flags, keys, (uint32_t)n, t.block_cnt, t.split_bit, t.leaf_start,
                                                  t.pt_leaf, t.d_meta, t.visit, (int32_t*)t.nodes, nw);
    count_launch(1);
    if (ev_mid) cudaEventRecord(ev_mid, st);
    topology_boxes(dim, recs, n, t, st);
}

void build_topology(int dim, const uint64_t* keys, const int4* recs, int64_t n, int leaf_max, const TreeBufs& t,
                    cudaStream_t st, cudaEvent_t ev_mid) {
    const uint32_t un = (uint32_t)n;
    const int nw = dim == 2 ? (int)(sizeof(Node<2>) / 4) : (int)(sizeof(Node<3>) / 4);
    if (n <= 1) {
        // 0 or 1 point: a single (possibly empty) leaf; reuse the compaction kernel's
        // bookkeeping path with an empty pair range.
        cudaMemsetAsync(t.block_cnt, 0, 2 * sizeof(uint32_t), st);
        compact_kernel<<<1, TT, 0, st>>>(t.flags, keys, un, t.block_cnt, t.split_bit, t.leaf_start, t.pt_leaf, t.d_meta, t.visit,
                                         (int32_t*)t.nodes, nw);
        count_launch(1);
        if (ev_mid) cudaEventRecord(ev_mid, st);
        topology_boxes(dim, recs, n, t, st);
    } else {
        // one pass: flags + look-back numbering (status words and the tile counter live
        // in block_cnt, zeroed here)
        const uint32_t ntiles = (uint32_t)((n + TTILE2 - 1) / TTILE2);
        cudaMemsetAsync(t.block_cnt, 0, (ntiles + 1) * sizeof(uint32_t), st);
        const int nw = dim == 2 ? (int)(sizeof(Node<2>) / 4) : (int)(sizeof(Node<3>) / 4);
        topo_kernel<<<ntiles, TT, 0, st>>>(keys, un, leaf_max, t.block_cnt, ntiles, t.split_bit, t.leaf_start, t.pt_leaf,
                                           t.d_meta, t.visit, (int32_t*)t.nodes, nw);
        count_launch(1);
        if (ev_mid) cudaEventRecord(ev_mid, st);
        topology_boxes(dim, recs, n, t, st);
    }
}

static void topology_boxes(int dim, const int4* recs, int64_t n, const TreeBufs& t, cudaStream_t st) {
    // one block per BW-leaf window; leaves <= max(n, 1) (windows past the last leaf exit
    // at once, before touching the node-indexed buffers)
    int grid = (int)std::max<int64_t>(1, (std::max<int64_t>(n, 1) + BW - 1) / BW);
    count_launch(1);
    if (dim == 2)
        bottom_up_kernel<2><<<grid, BW, 0, st>>>(recs, t.leaf_start, t.split_bit, t.d_meta, (Node<2>*)t.nodes,
                                                  t.leaf_parent, t.visit, t.range, t.pos_range);
    else
        bottom_up_kernel<3><<<grid, BW, 0, st>>>(recs, t.leaf_start, t.split_bit, t.d_meta, (Node<3>*)t.nodes,
                                                  t.leaf_parent, t.visit, t.range, t.pos_range);
}

}  // namespace zd
