// sort.cu — K1 Morton encode + K2 one-sweep LSD radix sort of (key, id) + K3 records.
//
// PAPER.md P:235 (§2 "Construction": "We then sort the points by the Morton
// order"), P:416 (Thm 2.1: "a parallel radix sort can be used").
// B200 design (not the paper's): 8 passes of 8-bit digits over 64-bit keys; one
// up-front histogram kernel computes all 8 digit histograms while encoding (and
// range-checking) the points; each pass is ONE kernel that ranks a 2816-key tile
// with warp-level match, publishes its per-digit counts, resolves its global
// offsets by decoupled look-back over predecessor tiles (dynamic tile ids, so
// every predecessor is resident or done), stages the tile in shared memory in
// digit order and scatters runs of equal digits coalesced.  Pass 1 reads the
// int32 points directly (encode fused, ids = iota); the last pass decodes the
// coordinates from the key and writes the 16-byte records (K3 fused).
#include <cstdio>
#include <cstdlib>

#include <cuda/atomic>

#include "common.cuh"
#include "internal.h"

namespace zd {

namespace {

constexpr int ST = 256;              // threads per tile
#ifndef ZD_SORT_SI
#define ZD_SORT_SI 13
#endif
#ifndef ZD_SORT_MINB
#define ZD_SORT_MINB 4
#endif
constexpr int SI = ZD_SORT_SI;       // keys per thread
constexpr int STILE = ST * SI;       // 2816 keys per tile (256 threads x 11)
constexpr int SW = ST / 32;          // warps
constexpr int WITEMS = 32 * SI;      // contiguous keys per warp
constexpr int NPASS = 8;
constexpr uint32_t VAL_MASK = (1u << 30) - 1;
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_INC = 2u << 30;

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    return cuda::atomic_ref<const uint32_t, cuda::thread_scope_device>(*p).load(cuda::memory_order_relaxed);
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    cuda::atomic_ref<uint32_t, cuda::thread_scope_device>(*p).store(v, cuda::memory_order_relaxed);
}

// Random shift applied after the range check: sh = (sx, sy, sz, mode), mode 0
// none, 2: 2D (31-bit shifted axes, 62-bit keys), 3: 3D (22-bit shifted axes; the key
// interleaves their levels 21..1 = 63 bits, reading R31).
template <int DIM>
__device__ __forceinline__ uint64_t shifted_key(int x, int y, int z, int4 sh) {
    if (DIM == 2) return morton<2>(x + sh.x, y + sh.y, 0);
    if (sh.w == 3) return morton<3>((x + sh.x) >> 1, (y + sh.y) >> 1, (z + sh.z) >> 1);
    return morton<3>(x, y, z);
}

// Range check in the universe box, then the key of the (shifted) point.
template <int DIM>
__device__ __forceinline__ uint64_t load_key_from_points(const int32_t* __restrict__ pts, uint32_t i, bool& bad,
                                                         int4 sh) {
    const int32_t* p = pts + (size_t)i * DIM;
    int x = __ldg(p), y = __ldg(p + 1), z = DIM == 3 ? __ldg(p + 2) : 0;
    bad |= !in_universe<DIM>(x, y, z);
    return shifted_key<DIM>(x, y, z, sh);
}

// Up-front histogram of the digits P0..7 (+ range validation): the truncated sorts
// never run passes 0..P0-1, and the shared-memory atomics (one per key and digit)
// bound this kernel.
template <int DIM, int P0>
__global__ void __launch_bounds__(256) hist_kernel(const int32_t* __restrict__ pts, uint32_t n,
                                                   uint32_t* __restrict__ g_hist, int* __restrict__ invalid, int4 sh2,
                                                   uint64_t* __restrict__ keys_out) {
    constexpr int NP = NPASS - P0;
    __shared__ uint32_t sh[NP][256];
    for (int i = threadIdx.x; i < NP * 256; i += 256) (&sh[0][0])[i] = 0;
    __syncthreads();
    bool bad = false;
    for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
        uint64_t key = load_key_from_points<DIM>(pts, i, bad, sh2);
        keys_out[i] = key;   // the first pass reads these instead of re-encoding
#pragma unroll
        for (int p = P0; p < NPASS; ++p) atomicAdd(&sh[p - P0][(key >> (8 * p)) & 255], 1u);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(invalid, 1);
    for (int i = threadIdx.x; i < NP * 256; i += 256) {
        uint32_t v = (&sh[0][0])[i];
        if (v) atomicAdd(g_hist + P0 * 256 + i, v);
    }
}

__global__ void __launch_bounds__(256) scan_hist_kernel(const uint32_t* __restrict__ g_hist, uint32_t* __restrict__ offs) {
    __shared__ uint32_t s_warp[32];
    const int p = blockIdx.x;   // one block per digit
    uint32_t v = g_hist[p * 256 + threadIdx.x];
    offs[p * 256 + threadIdx.x] = block_exclusive_scan<256>(v, s_warp, nullptr);
}

// MODE 0: first pass (encode points), 1: middle pass, 2: last pass (write records).
template <int DIM, int MODE>
__global__ void __launch_bounds__(ST, ZD_SORT_MINB) onesweep_kernel(
    const int32_t* __restrict__ pts, const uint64_t* __restrict__ keys_in, const uint32_t* __restrict__ ids_in,
    uint64_t* __restrict__ keys_out, uint32_t* __restrict__ ids_out, int4* __restrict__ recs_out,
    uint32_t n, int shift, uint32_t id_base, const uint32_t* __restrict__ digit_offs,
    uint32_t* status, uint32_t* tile_counter, int4 psh) {
    __shared__ union {
        uint32_t hist[SW][256];
        uint64_t keys[STILE];
    } u;
    __shared__ uint32_t s_ids[STILE];
    __shared__ uint32_t s_start[256];
    __shared__ uint32_t s_glob[256];
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
    for (int i = tid; i < SW * 256; i += ST) (&u.hist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t tile_base = tile * STILE;
    const uint32_t base = tile_base + w * WITEMS + lane;

    // ---- load (warp-blocked: warp w owns 480 contiguous keys, so rank order = input order)
    uint64_t key[SI];
    uint32_t id[SI];
    bool bad = false;
#pragma unroll
    for (int j = 0; j < SI; ++j) {
        uint32_t idx = base + j * 32;
        if (idx < n) {
            if (MODE == 0) {
                key[j] = keys_in[idx];   // encoded (and range-checked) by hist_kernel
                id[j] = id_base + idx;
            } else {
                key[j] = keys_in[idx];
                id[j] = ids_in[idx];
            }
        } else {
            key[j] = ~0ull;   // sorts last within the tile; never written out
            id[j] = 0;
        }
    }

    // ---- warp-level ranking: peers with the same digit via match.any
    uint32_t loc[SI];
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < SI; ++j) {
        // the lowest lane of each digit group bumps the warp-private counter by the
        // group size (shared-memory atomic: same-address atomics of one warp are
        // applied in issue order, so key j's group precedes key j+1's — stable) and
        // broadcasts the old value; no __syncwarp chain between the SI keys
        const uint32_t d = (uint32_t)(key[j] >> shift) & 255u;
        // lanes with the same digit: 8 ballots (one per digit bit) instead of the
        // slow match.any
        uint32_t peers = 0xffffffffu;
#pragma unroll
        for (int bit = 0; bit < 8; ++bit) {
            const bool on = (d >> bit) & 1u;
            const uint32_t bv = __ballot_sync(0xffffffffu, on);
            peers &= on ? bv : ~bv;
        }
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (lane == leader) old = atomicAdd(&u.hist[w][d], (uint32_t)__popc(peers));
        old = __shfl_sync(0xffffffffu, old, leader);
        loc[j] = old + __popc(peers & lt_mask);
    }
    __syncthreads();

    // ---- per-digit tile counts (thread = digit) and warp prefixes
    uint32_t cnt = 0;
#pragma unroll
    for (int ww = 0; ww < SW; ++ww) {
        uint32_t c = u.hist[ww][tid];
        u.hist[ww][tid] = cnt;
        cnt += c;
    }
    uint32_t* my_status = status + (size_t)tile * 256 + tid;
    if (tile == 0) st_relaxed(my_status, FLAG_INC | cnt);
    else st_relaxed(my_status, FLAG_AGG | cnt);

    const uint32_t start = block_exclusive_scan<ST>(cnt, s_warp, nullptr);
    s_start[tid] = start;

    // ---- decoupled look-back (one digit per thread)
    // Windowed: LB predecessors' status words are loaded at once (independent loads,
    // one round trip) and folded nearest-first until an inclusive prefix; an
    // unpublished predecessor ends the window and is re-read.  Tile 0 is inclusive,
    // so the walk never passes it.
    uint32_t excl = 0;
    if (tile > 0) {
        constexpr int LB = 8;
        int64_t t = (int64_t)tile - 1;
        while (true) {
            // spin on the nearest unread predecessor alone, then fold a window
            uint32_t v0;
            do { v0 = ld_relaxed(status + (size_t)t * 256 + tid); } while ((v0 & ~VAL_MASK) == 0);
            excl += v0 & VAL_MASK;
            if ((v0 & ~VAL_MASK) == FLAG_INC) break;
            --t;
            uint32_t v[LB];
#pragma unroll
            for (int k = 0; k < LB; ++k)
                v[k] = (t - k >= 0) ? ld_relaxed(status + (size_t)(t - k) * 256 + tid) : (FLAG_INC | 0u);
            bool done = false;
            int used = 0;
#pragma unroll
            for (int k = 0; k < LB; ++k) {
                if (done || used < k) continue;                    // stopped earlier in this window
                if ((v[k] & ~VAL_MASK) == 0) continue;             // not published: spin on it next
                excl += v[k] & VAL_MASK;
                used = k + 1;
                if ((v[k] & ~VAL_MASK) == FLAG_INC) done = true;
            }
            if (done) break;
            t -= used;
        }
        st_relaxed(my_status, FLAG_INC | (excl + cnt));
    }
    s_glob[tid] = digit_offs[tid] + excl - start;
    __syncthreads();

#pragma unroll
    for (int j = 0; j < SI; ++j) {
        uint32_t d = (uint32_t)(key[j] >> shift) & 255u;
        loc[j] += s_start[d] + u.hist[w][d];
    }
    __syncthreads();   // all hist reads done before the union is reused for keys
#pragma unroll
    for (int j = 0; j < SI; ++j) {
        u.keys[loc[j]] = key[j];
        s_ids[loc[j]] = id[j];
    }
    __syncthreads();

    // ---- scatter in digit order: runs of equal digits go to consecutive addresses
    const uint32_t valid = min((uint32_t)STILE, n - tile_base);
    for (uint32_t i = tid; i < valid; i += ST) {
        uint64_t k = u.keys[i];
        uint32_t d = (uint32_t)(k >> shift) & 255u;
        uint32_t dest = s_glob[d] + i;
        ZD_DCHECK(dest < n);
        keys_out[dest] = k;
        if (MODE == 2) {
            if (DIM == 3 && psh.w == 3) {
                // 3D shift: the key drops each coordinate's lowest bit, so the record
                // comes from the input point (ids of a sort are id_base + input index)
                const uint32_t id = s_ids[i];
                ZD_DCHECK(id - id_base < n);
                const int32_t* p = pts + (size_t)(id - id_base) * 3;
                recs_out[dest] = make_int4(__ldg(p) + psh.x, __ldg(p + 1) + psh.y, __ldg(p + 2) + psh.z, (int)id);
            } else {
                recs_out[dest] = decode_rec<DIM>(k, (int)s_ids[i]);
            }
        }
        else ids_out[dest] = s_ids[i];
    }
    (void)bad;
}

// Truncated sort (large builds): the LSD passes cover only the digits above bit
// kTruncBits, leaving runs of keys that agree on bits >= kTruncBits in input (= id)
// order; each element then finds its run and its rank in it by (key, id) and is
// written to its final place, with its record.  Runs are short for real inputs (at 10M
// 3D points the 39-bit prefix is shared by ~1 point on average, by ~4-10 at the
// centre of the Plummer sphere); a run longer than kTruncRun sets *fail and the
// caller redoes the sort with all 8 passes (checked at the build's one sync).
constexpr int kTruncBits = 24;      // digits 3..7 sorted: 5 passes instead of 8
constexpr uint32_t kTruncRun = 64;  // longest run resolved by the rank fixup
template <int DIM>
__global__ void __launch_bounds__(256) trunc_fixup_kernel(const uint64_t* __restrict__ keys_in,
                                                          const uint32_t* __restrict__ ids_in, uint32_t n,
                                                          uint64_t* __restrict__ keys_out, int4* __restrict__ recs_out,
                                                          const int32_t* __restrict__ pts, uint32_t id_base, int4 psh,
                                                          int* __restrict__ fail) {
    const uint32_t i = blockIdx.x * 256 + threadIdx.x;
    if (i >= n) return;
    const uint64_t k = keys_in[i];
    const uint32_t id = ids_in[i];
    const uint64_t pre = k >> kTruncBits;
    uint32_t lo = i, hi = i + 1;
    while (lo > 0 && (__ldg(keys_in + lo - 1) >> kTruncBits) == pre) {
        if (i - --lo >= kTruncRun) { atomicOr(fail, 1); return; }
    }
    while (hi < n && (__ldg(keys_in + hi) >> kTruncBits) == pre) {
        if (++hi - i > kTruncRun) { atomicOr(fail, 1); return; }
    }
    uint32_t rank = 0;
    for (uint32_t j = lo; j < hi; ++j) {
        const uint64_t kj = __ldg(keys_in + j);
        const uint32_t ij = __ldg(ids_in + j);
        rank += (kj < k || (kj == k && ij < id)) ? 1u : 0u;   // ids are distinct: j == i never counts
    }
    const uint32_t dest = lo + rank;
    ZD_DCHECK(dest < n);
    keys_out[dest] = k;
    if (DIM == 3 && psh.w == 3) {
        const int32_t* p = pts + (size_t)(id - id_base) * 3;
        recs_out[dest] = make_int4(__ldg(p) + psh.x, __ldg(p + 1) + psh.y, __ldg(p + 2) + psh.z, (int)id);
    } else {
        recs_out[dest] = decode_rec<DIM>(k, (int)id);
    }
}

// Small sorts (n <= kSmallSort, e.g. the batch of a small insert): one block ranks each
// key by counting the (key, index) pairs below it — one launch instead of the
// histogram, scan and eight one-sweep passes (which cost ~0.1 ms even for one key).
template <int DIM>
__global__ void __launch_bounds__(kSmallSort) small_sort_kernel(const int32_t* __restrict__ pts, uint32_t n, uint32_t id_base,
                                                                int4 psh, uint64_t* __restrict__ keys_out,
                                                                int4* __restrict__ recs_out, int* __restrict__ invalid) {
    __shared__ uint64_t s_key[kSmallSort];
    const uint32_t i = threadIdx.x;
    bool bad = false;
    uint64_t k = ~0ull;
    if (i < n) k = load_key_from_points<DIM>(pts, i, bad, psh);
    s_key[i] = k;
    if (__syncthreads_or(bad) && i == 0) atomicOr(invalid, 1);
    if (i >= n) return;
    uint32_t rank = 0;   // stable: equal keys keep input (= id) order
    for (uint32_t j = 0; j < n; ++j) {
        const uint64_t kj = s_key[j];
        rank += (kj < k || (kj == k && j < i)) ? 1u : 0u;
    }
    keys_out[rank] = k;
    const uint32_t id = id_base + i;
    if (DIM == 3 && psh.w == 3) {
        const int32_t* p = pts + (size_t)i * 3;
        recs_out[rank] = make_int4(__ldg(p) + psh.x, __ldg(p + 1) + psh.y, __ldg(p + 2) + psh.z, (int)id);
    } else {
        recs_out[rank] = decode_rec<DIM>(k, (int)id);
    }
}

template <int DIM>
void sort_points_t(const int32_t* pts, int64_t n, uint32_t id_base, uint64_t* keys_out, int4* recs_out,
                   const SortScratch& s, int* d_invalid, int4 psh, cudaStream_t st, int* d_trunc_fail, bool approx) {
    const uint32_t un = (uint32_t)n;
    const size_t tiles = sort_tiles(n);
    uint32_t* hist = s.zero_block;
    uint32_t* counters = hist + NPASS * 256;
    uint32_t* status = counters + NPASS;
    // development aid: ZD_SORT_PROFILE=1 prints per-kernel device times of each sort
    static const bool prof = std::getenv("ZD_SORT_PROFILE") != nullptr;
    cudaEvent_t pev[NPASS + 4] = {};
    int npev = 0;
    auto mark = [&]() {
        if (!prof) return;
        cudaEventCreate(&pev[npev]);
        cudaEventRecord(pev[npev++], st);
    };
    mark();
    if (approx || d_trunc_fail) {
        // histograms and tile counters, then the look-back words of the passes that run
        constexpr size_t P0 = kTruncBits / 8;
        cudaMemsetAsync(s.zero_block, 0, (NPASS * 256 + NPASS) * sizeof(uint32_t), st);
        cudaMemsetAsync(status + P0 * tiles * 256, 0, (NPASS - P0) * tiles * 256 * sizeof(uint32_t), st);
    } else {
        cudaMemsetAsync(s.zero_block, 0, sort_zero_words(n) * sizeof(uint32_t), st);
    }
    mark();
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int hb = (int)std::min<size_t>((size_t)sms * 8, (n + 255) / 256);
    if (approx || d_trunc_fail)
        hist_kernel<DIM, kTruncBits / 8><<<hb, 256, 0, st>>>(pts, un, hist, d_invalid, psh, s.k[1]);
    else
        hist_kernel<DIM, 0><<<hb, 256, 0, st>>>(pts, un, hist, d_invalid, psh, s.k[1]);
    scan_hist_kernel<<<NPASS, 256, 0, st>>>(hist, s.offs);
    mark();
    if (approx) {
        // order only by key bits 24..63 (digits 3..7); keys sharing those bits stay in
        // input order — enough for the Morton locality of query batches
        constexpr int P0 = kTruncBits / 8;
        count_launch(2 + (NPASS - P0));
        for (int p = P0; p < NPASS; ++p) {
            const int q = p - P0;
            uint32_t* stp = status + (size_t)p * tiles * 256;
            const uint32_t* off = s.offs + p * 256;
            if (q == 0)
                onesweep_kernel<DIM, 0><<<tiles, ST, 0, st>>>(pts, s.k[1], nullptr, s.k[0], s.v[0], nullptr, un, 8 * p,
                                                              id_base, off, stp, counters + p, psh);
            else if (p < NPASS - 1)
                onesweep_kernel<DIM, 1><<<tiles, ST, 0, st>>>(nullptr, s.k[(q - 1) & 1], s.v[(q - 1) & 1], s.k[q & 1],
                                                              s.v[q & 1], nullptr, un, 8 * p, 0, off, stp, counters + p,
                                                              psh);
            else
                onesweep_kernel<DIM, 2><<<tiles, ST, 0, st>>>(pts, s.k[(q - 1) & 1], s.v[(q - 1) & 1], keys_out,
                                                              nullptr, recs_out, un, 8 * p, id_base, off, stp,
                                                              counters + p, psh);
            mark();
        }
    } else if (d_trunc_fail) {
        // digits 3..7 (bits 24..63), then the rank fixup of equal-prefix runs
        constexpr int P0 = kTruncBits / 8;
        count_launch(2 + (NPASS - P0) + 1);
        for (int p = P0; p < NPASS; ++p) {
            const int q = p - P0;   // ping-pong index
            uint32_t* stp = status + (size_t)p * tiles * 256;
            const uint32_t* off = s.offs + p * 256;
            if (q == 0)
                onesweep_kernel<DIM, 0><<<tiles, ST, 0, st>>>(pts, s.k[1], nullptr, s.k[0], s.v[0], nullptr, un, 8 * p,
                                                              id_base, off, stp, counters + p, psh);
            else
                onesweep_kernel<DIM, 1><<<tiles, ST, 0, st>>>(nullptr, s.k[(q - 1) & 1], s.v[(q - 1) & 1], s.k[q & 1],
                                                              s.v[q & 1], nullptr, un, 8 * p, 0, off, stp, counters + p,
                                                              psh);
            mark();
        }
        const int qlast = NPASS - 1 - P0;
        trunc_fixup_kernel<DIM><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
            s.k[qlast & 1], s.v[qlast & 1], un, keys_out, recs_out, pts, id_base, psh, d_trunc_fail);
        mark();
    } else {
    count_launch(2 + NPASS);
    for (int p = 0; p < NPASS; ++p) {
        uint32_t* stp = status + (size_t)p * tiles * 256;
        const uint32_t* off = s.offs + p * 256;
        if (p == 0)
            onesweep_kernel<DIM, 0><<<tiles, ST, 0, st>>>(pts, s.k[1], nullptr, s.k[0], s.v[0], nullptr, un, 0,
                                                          id_base, off, stp, counters + p, psh);
        else if (p < NPASS - 1)
            onesweep_kernel<DIM, 1><<<tiles, ST, 0, st>>>(nullptr, s.k[(p - 1) & 1], s.v[(p - 1) & 1], s.k[p & 1],
                                                          s.v[p & 1], nullptr, un, 8 * p, 0, off, stp, counters + p, psh);
        else
            onesweep_kernel<DIM, 2><<<tiles, ST, 0, st>>>(pts, s.k[(p - 1) & 1], s.v[(p - 1) & 1], keys_out,
                                                          nullptr, recs_out, un, 8 * p, id_base, off, stp, counters + p,
                                                          psh);
        mark();
    }
    }
    if (prof) {
        cudaEventSynchronize(pev[npev - 1]);
        fprintf(stderr, "sort n=%lld:", (long long)n);
        for (int i = 1; i < npev; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, pev[i - 1], pev[i]);
            fprintf(stderr, " %.1f", ms * 1e3f);
        }
        fprintf(stderr, " us\n");
        for (int i = 0; i < npev; ++i) cudaEventDestroy(pev[i]);
    }
}

}  // namespace

void sort_points_small(int dim, const int32_t* pts, int64_t n, uint32_t id_base, uint64_t* keys_out, int4* recs_out,
                       int* d_invalid, cudaStream_t st, const int32_t* shift2) {
    if (n <= 0) return;
    const int4 psh = shift2 ? make_int4(shift2[0], shift2[1], dim == 3 ? shift2[2] : 0, dim)
                            : make_int4(0, 0, 0, 0);
    count_launch(1);
    if (dim == 2) small_sort_kernel<2><<<1, kSmallSort, 0, st>>>(pts, (uint32_t)n, id_base, psh, keys_out, recs_out, d_invalid);
    else small_sort_kernel<3><<<1, kSmallSort, 0, st>>>(pts, (uint32_t)n, id_base, psh, keys_out, recs_out, d_invalid);
}

size_t sort_tiles(int64_t n) { return (size_t)((n + STILE - 1) / STILE); }
size_t sort_zero_words(int64_t n) { return NPASS * 256 + NPASS + (size_t)NPASS * sort_tiles(n) * 256; }

void sort_points(int dim, const int32_t* pts, int64_t n, uint32_t id_base, uint64_t* keys_out, int4* recs_out,
                 const SortScratch& s, int* d_invalid, cudaStream_t st, const int32_t* shift2, int* d_trunc_fail,
                 bool approx) {
    if (n <= 0) return;
    const int4 psh = shift2 ? make_int4(shift2[0], shift2[1], dim == 3 ? shift2[2] : 0, dim)
                            : make_int4(0, 0, 0, 0);
    if (dim == 2) sort_points_t<2>(pts, n, id_base, keys_out, recs_out, s, d_invalid, psh, st, d_trunc_fail, approx);
    else sort_points_t<3>(pts, n, id_base, keys_out, recs_out, s, d_invalid, psh, st, d_trunc_fail, approx);
}

}  // namespace zd
