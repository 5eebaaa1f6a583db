// update.cu — K7-K9 batch insert / delete support kernels.
//
// PAPER.md Alg. 4 batchInsert routes a Morton-sorted batch down the
// tree by each node's split bit; with empty cuts skipped that routing can
// place a key in a subtree whose Morton cell does not contain it (SURVEY §8(c)
// reading 17), so this build keeps the tree canonical instead: the sorted batch is
// MERGED into the sorted (key, record) arrays (merge path; equal keys keep the
// older, smaller id first) and the topology + boxes are rebuilt from the merged
// arrays (tree.cu).  Deletion ("almost identical") clears the ids in an
// alive bitset and stably compacts the sorted arrays.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace zd {

namespace {

int num_sms() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

__global__ void __launch_bounds__(256) validate_kernel(const int32_t* __restrict__ v, int64_t count, uint32_t lim,
                                                       int* __restrict__ invalid) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < count; i += (int64_t)gridDim.x * 256)
        bad |= (uint32_t)__ldg(v + i) >= lim;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(invalid, 1);
}

constexpr int MT = 256;
constexpr int MI = 8;
constexpr int MTILE = MT * MI;   // outputs per block

// merge path: number of A elements among the first `diag` outputs (A wins ties)
__device__ __forceinline__ int64_t merge_split(const uint64_t* __restrict__ ka, int64_t n, const uint64_t* __restrict__ kb,
                                               int64_t m, int64_t diag) {
    int64_t lo = max((int64_t)0, diag - m), hi = min(diag, n);
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(ka + mid) <= __ldg(kb + diag - 1 - mid)) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Block-tiled merge path: a block owns MTILE consecutive outputs; it stages the two
// input key runs in shared memory, each thread merges MI outputs there and records
// their sources, and the block then writes keys and records coalesced.
__global__ void __launch_bounds__(MT) merge_kernel(const uint64_t* __restrict__ ka, const int4* __restrict__ ra, int64_t n,
                                                   const uint64_t* __restrict__ kb, const int4* __restrict__ rb, int64_t m,
                                                   uint64_t* __restrict__ ko, int4* __restrict__ ro) {
    __shared__ uint64_t s_key[MTILE];
    __shared__ int32_t s_src[MTILE];   // >= 0: A offset in the tile; < 0: ~B offset
    __shared__ int64_t s_split[2];
    const int64_t tot = n + m;
    const int64_t d0 = (int64_t)blockIdx.x * MTILE;
    const int64_t d1 = min(d0 + MTILE, tot);
    if (threadIdx.x < 2) s_split[threadIdx.x] = merge_split(ka, n, kb, m, threadIdx.x ? d1 : d0);
    __syncthreads();
    const int64_t a0 = s_split[0], a1 = s_split[1];
    const int64_t b0 = d0 - a0, b1 = d1 - a1;
    const int na = (int)(a1 - a0), nb = (int)(b1 - b0);
    for (int i = threadIdx.x; i < na + nb; i += MT)
        s_key[i] = i < na ? __ldg(ka + a0 + i) : __ldg(kb + b0 + (i - na));
    __syncthreads();
    // this thread's outputs [t0, t0 + MI) within the tile
    const int t0 = threadIdx.x * MI;
    if (t0 < na + nb) {
        int lo = max(0, t0 - nb), hi = min(t0, na);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s_key[mid] <= s_key[na + t0 - 1 - mid]) lo = mid + 1; else hi = mid;
        }
        int ia = lo, ib = t0 - lo;
#pragma unroll
        for (int t = 0; t < MI; ++t) {
            const int o = t0 + t;
            if (o >= na + nb) break;
            const bool take_a = ib >= nb || (ia < na && s_key[ia] <= s_key[na + ib]);
            s_src[o] = take_a ? ia++ : ~(ib++);
        }
    }
    __syncthreads();
    for (int o = threadIdx.x; o < na + nb; o += MT) {
        const int sidx = s_src[o];
        ZD_DCHECK(d0 + o < tot && (sidx >= 0 ? sidx < na : ~sidx < nb));
        ko[d0 + o] = sidx >= 0 ? s_key[sidx] : s_key[na + ~sidx];
        ro[d0 + o] = sidx >= 0 ? __ldg(ra + a0 + sidx) : __ldg(rb + b0 + ~sidx);
    }
}

__global__ void __launch_bounds__(256) set_alive_kernel(uint32_t* alive, int64_t first, int64_t count) {
    const int64_t end = first + count;
    for (int64_t w = (first >> 5) + (int64_t)blockIdx.x * 256 + threadIdx.x; (w << 5) < end;
         w += (int64_t)gridDim.x * 256) {
        const int64_t b0 = w << 5;
        uint32_t mask = 0xffffffffu;
        if (b0 < first) mask &= 0xffffffffu << (first - b0);
        if (b0 + 32 > end) mask &= 0xffffffffu >> (b0 + 32 - end);
        atomicOr(alive + w, mask);
    }
}

__global__ void __launch_bounds__(256) mark_deleted_kernel(uint32_t* alive, int64_t id_cap, const int32_t* __restrict__ ids,
                                                           int64_t m, unsigned long long* count) {
    unsigned long long c = 0;
    for (int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x; t < m; t += (int64_t)gridDim.x * 256) {
        const int32_t id = __ldg(ids + t);
        if (id < 0 || id >= id_cap) continue;               // absent id: skipped
        const uint32_t bit = 1u << (id & 31);
        const uint32_t old = atomicAnd(alive + (id >> 5), ~bit);
        c += (old & bit) ? 1 : 0;                           // dead or duplicate: skipped
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

constexpr int CT = 256;
constexpr int CPI = 8;
constexpr int CTILE = CT * CPI;

__device__ __forceinline__ bool is_alive(const uint32_t* alive, int32_t id) {
    return (__ldg(alive + (id >> 5)) >> (id & 31)) & 1u;
}

__global__ void __launch_bounds__(CT) compact_count_kernel(const uint32_t* __restrict__ alive, const int4* __restrict__ ri,
                                                           int64_t n, uint32_t* __restrict__ block_cnt) {
    __shared__ uint32_t s_warp[32];
    const int64_t base = (int64_t)blockIdx.x * CTILE + threadIdx.x;
    uint32_t c = 0;
#pragma unroll
    for (int t = 0; t < CPI; ++t) {
        const int64_t i = base + t * CT;
        if (i < n) c += is_alive(alive, __ldg(&ri[i].w));
    }
    uint32_t tot;
    block_exclusive_scan<CT>(c, s_warp, &tot);
    if (threadIdx.x == 0) block_cnt[blockIdx.x] = tot;
}

// Stable compaction of one CTILE tile: element (j, t) = base + j*CT + t is read
// coalesced; its output rank = kept elements before it in (j, warp, lane) order, from
// per-(j, warp) ballot counts scanned by one warp.
__global__ void __launch_bounds__(CT) compact_write_kernel(const uint32_t* __restrict__ alive, const uint64_t* __restrict__ ki,
                                                           const int4* __restrict__ ri, int64_t n,
                                                           const uint32_t* __restrict__ block_off,
                                                           uint64_t* __restrict__ ko, int4* __restrict__ ro) {
    constexpr int NW = CT / 32;
    __shared__ uint32_t s_cnt[CPI * NW];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * CTILE + threadIdx.x;
    int4 r[CPI];
    uint32_t bal[CPI];
#pragma unroll
    for (int j = 0; j < CPI; ++j) {
        const int64_t i = base + (int64_t)j * CT;
        bool keep = false;
        if (i < n) {
            r[j] = __ldg(ri + i);
            keep = is_alive(alive, r[j].w);
        }
        bal[j] = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_cnt[j * NW + w] = __popc(bal[j]);
    }
    __syncthreads();
    if (w == 0) {   // exclusive scan of the CPI*NW counts (j-major, then warp)
        uint32_t carry = 0;
        for (int c0 = 0; c0 < CPI * NW; c0 += 32) {
            const uint32_t v = c0 + lane < CPI * NW ? s_cnt[c0 + lane] : 0u;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (c0 + lane < CPI * NW) s_cnt[c0 + lane] = carry + x - v;
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
    }
    __syncthreads();
    const uint32_t off = block_off[blockIdx.x];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < CPI; ++j) {
        if ((bal[j] >> lane) & 1u) {
            const uint32_t o = off + s_cnt[j * NW + w] + __popc(bal[j] & lt);
            ZD_DCHECK(o < n);
            ko[o] = __ldg(ki + base + (int64_t)j * CT);
            ro[o] = r[j];
        }
    }
}

constexpr int RT = 256;   // one 32-id word per thread

__global__ void __launch_bounds__(RT) rank_count_kernel(const uint32_t* __restrict__ alive, int64_t words,
                                                        uint32_t* __restrict__ block_cnt) {
    __shared__ uint32_t s_warp[32];
    const int64_t w = (int64_t)blockIdx.x * RT + threadIdx.x;
    const uint32_t c = w < words ? __popc(__ldg(alive + w)) : 0u;
    uint32_t tot;
    block_exclusive_scan<RT>(c, s_warp, &tot);
    if (threadIdx.x == 0) block_cnt[blockIdx.x] = tot;
}

// One block = the 256 alive words (8192 ids) of rank_count_kernel's block; ids are
// then visited one per thread (coalesced row_of_id writes).
__global__ void __launch_bounds__(RT) rank_write_kernel(const uint32_t* __restrict__ alive, int64_t words, int64_t id_cap,
                                                        const uint32_t* __restrict__ block_off,
                                                        int32_t* __restrict__ row_of_id, int32_t* __restrict__ live_ids) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_bits[RT], s_pre[RT];
    const int64_t w = (int64_t)blockIdx.x * RT + threadIdx.x;
    const uint32_t bits = w < words ? __ldg(alive + w) : 0u;
    s_bits[threadIdx.x] = bits;
    s_pre[threadIdx.x] = block_off[blockIdx.x] + block_exclusive_scan<RT>(__popc(bits), s_warp, nullptr);
    __syncthreads();
    const int64_t id0 = (int64_t)blockIdx.x * RT * 32;
    for (int t = threadIdx.x; t < RT * 32; t += RT) {
        const int64_t id = id0 + t;
        if (id >= id_cap) break;
        const uint32_t b = s_bits[t >> 5];
        const int bit = t & 31;
        if ((b >> bit) & 1u) {
            const uint32_t r = s_pre[t >> 5] + __popc(b & ((1u << bit) - 1u));
            row_of_id[id] = (int32_t)r;
            live_ids[r] = (int32_t)id;
        } else {
            row_of_id[id] = -1;
        }
    }
}

}  // namespace

void validate_points(int dim, const int32_t* pts, int64_t m, int* d_invalid, cudaStream_t st) {
    const int64_t count = m * dim;
    if (count <= 0) return;
    const uint32_t lim = 1u << (dim == 2 ? Dim<2>::B : Dim<3>::B);
    const int grid = (int)std::min<int64_t>((int64_t)num_sms() * 4, (count + 255) / 256);
    validate_kernel<<<grid, 256, 0, st>>>(pts, count, lim, d_invalid);
    count_launch(1);
}

void merge_sorted(const uint64_t* ka, const int4* ra, int64_t n, const uint64_t* kb, const int4* rb, int64_t m,
                  uint64_t* ko, int4* ro, cudaStream_t st) {
    const int64_t tot = n + m;
    if (tot <= 0) return;
    merge_kernel<<<(unsigned)((tot + MTILE - 1) / MTILE), MT, 0, st>>>(ka, ra, n, kb, rb, m, ko, ro);
    count_launch(1);
}

void set_alive_range(uint32_t* alive, int64_t first, int64_t count, cudaStream_t st) {
    if (count <= 0) return;
    const int64_t words = ((first + count + 31) >> 5) - (first >> 5);
    const int grid = (int)std::min<int64_t>((int64_t)num_sms() * 4, (words + 255) / 256);
    set_alive_kernel<<<grid, 256, 0, st>>>(alive, first, count);
    count_launch(1);
}

void mark_deleted(uint32_t* alive, int64_t id_cap, const int32_t* ids, int64_t m, unsigned long long* d_count,
                  cudaStream_t st) {
    if (m <= 0) return;
    const int grid = (int)std::min<int64_t>((int64_t)num_sms() * 4, (m + 255) / 256);
    mark_deleted_kernel<<<grid, 256, 0, st>>>(alive, id_cap, ids, m, d_count);
    count_launch(1);
}

size_t compact_blocks(int64_t n) { return (size_t)std::max<int64_t>(1, (n + CTILE - 1) / CTILE); }

void compact_alive(const uint32_t* alive, const uint64_t* ki, const int4* ri, int64_t n, uint64_t* ko, int4* ro,
                   uint32_t* block_cnt, cudaStream_t st) {
    if (n <= 0) return;
    const size_t nb = compact_blocks(n);
    compact_count_kernel<<<nb, CT, 0, st>>>(alive, ri, n, block_cnt);
    scan_blocks_kernel<<<1, 1024, 0, st>>>(block_cnt, (uint32_t)nb);
    compact_write_kernel<<<nb, CT, 0, st>>>(alive, ki, ri, n, block_cnt, ko, ro);
    count_launch(3);
}

size_t rank_blocks(int64_t id_cap) { return (size_t)std::max<int64_t>(1, (((id_cap + 31) >> 5) + RT - 1) / RT); }

void rank_alive(const uint32_t* alive, int64_t id_cap, int32_t* row_of_id, int32_t* live_ids, uint32_t* block_cnt,
                cudaStream_t st) {
    if (id_cap <= 0) return;
    const int64_t words = (id_cap + 31) >> 5;
    const size_t nb = rank_blocks(id_cap);
    rank_count_kernel<<<nb, RT, 0, st>>>(alive, words, block_cnt);
    scan_blocks_kernel<<<1, 1024, 0, st>>>(block_cnt, (uint32_t)nb);
    rank_write_kernel<<<nb, RT, 0, st>>>(alive, words, id_cap, block_cnt, row_of_id, live_ids);
    count_launch(3);
}

}  // namespace zd
