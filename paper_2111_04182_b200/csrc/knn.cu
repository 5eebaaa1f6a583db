// knn.cu — K6 exact k-NN over the zd-tree: warp-cooperative ("packet") searchUp.
//
// PAPER.md: Alg. 3 searchUp calling Alg. 2 searchDown;
// leaf-based all-points search; bit-based location of external queries
// ("dynamic queries" P:183, App. B); queries walked in Morton order for
// locality.
//
// A warp owns a PACKET of 32 queries adjacent in Morton order (all-points: 32
// consecutive sorted positions; external: 32 consecutive Morton-sorted queries),
// whose leaves span lA..lB.  The warp runs ONE searchUp for the packet, each lane
// keeping its own k-best state:
//   1. scan leaves lA..lB (Alg. 3's leaf seed, for all lanes at once);
//   2. if lA != lB, searchDown over the rest of the subtree of X = lowest common
//      ancestor of lA and lB (leaves lA..lB skipped);
//   3. ascend from X: stop when EVERY lane's stop test holds at C (reading 9), else
//      searchDown the sibling of C, C = parent(C).
// searchDown is joint: a subtree is entered iff SOME lane's box distance is <= its
// bound (reading 8 per lane); nearer child first by lane majority (reading 10); the
// far child goes on a per-warp shared-memory stack with its box and is re-tested
// when popped.  Leaf points are staged through shared memory (coalesced 16-B loads,
// one record per lane) and broadcast to all lanes; a node whose children are both
// leaves is scanned as ONE contiguous span (its points are adjacent in sorted order).
//
// Scheduling: the first launch is a persistent grid of resident blocks; every warp takes
// the next packet in Morton order from a counter (packets differ ~2x in cost, so a
// fixed packet per warp left warps idle until their block's slowest finished).
//
// Per-lane k-best state (the warp never serialises on sorted insertions):
//   fa[K]  ascending list of the k smallest d2 seen so far, each rounded UP to fp32
//          (bf16 pairs for even K; ids ignored), kept with branch-free min/max;
//   U      = ceil(fa[K-1]) as int64: an upper bound on the exact k-th smallest d2 among
//          the candidates seen, hence on the final k-th distance; U never grows;
//   buf    (position, ru(d2)) of every candidate that had d2 <= U when seen.
// A subtree or candidate can hold a final neighbour only if its (box) d2 <= U, so
// pruning by "> U" (reading 8), stopping by "(m+1)^2 > U" (reading 9) and buffering
// by "d2 <= U" lose nothing.  The buffer is compacted by ru(d2) <= fa[K-1] (sound:
// rounding up is monotone), and at the end the ~k survivors are inserted exactly by
// (d2, id) (reading 14) into a register list.  Every lane's answer is exact: it sees
// a superset of what its own searchUp would see and drops a point only by its own
// sound rules; the (d2, id) order makes the answer unique.  Self is excluded by id
// (reading 13); short rows are padded with (-1, INT64_MAX) (reading 15).
#include <algorithm>
#include <climits>
#include <cstddef>

#include "common.cuh"
#include "internal.h"

namespace zd {

// Optional work counters (build with -DZD_KNN_STATS; see zd_knn_stats in zd.h).
#ifdef ZD_KNN_STATS
__device__ unsigned long long g_knn_stats[ZD_NSTATS];
#define ZD_STAT(i, v) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_knn_stats[i], (unsigned long long)(v)); } while (0)
#else
#define ZD_STAT(i, v) do { } while (0)
#endif

namespace {

template <int K>
struct KBest {
    int64_t d[K];
    int32_t i[K];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int s = 0; s < K; ++s) { d[s] = INT64_MAX; i[s] = -1; }
    }
    __device__ __forceinline__ bool accepts(int64_t cd, int32_t ci) const {
        return cd < d[K - 1] || (cd == d[K - 1] && ci < i[K - 1]);
    }
    // sorted insertion, branch-free over the unrolled register list
    __device__ __forceinline__ void insert(int64_t cd, int32_t ci) {
        bool lts = true;   // candidate < slot s  (true for s = K-1 by precondition)
#pragma unroll
        for (int s = K - 1; s > 0; --s) {
            const bool ltp = cd < d[s - 1] || (cd == d[s - 1] && ci < i[s - 1]);
            const int64_t nd = ltp ? d[s - 1] : (lts ? cd : d[s]);
            const int32_t ni = ltp ? i[s - 1] : (lts ? ci : i[s]);
            d[s] = nd;
            i[s] = ni;
            lts = ltp;
        }
        if (lts) { d[0] = cd; i[0] = ci; }
    }
};

template <int DIM>
struct Query {
    int c[3];
    int32_t id;   // excluded id; -1 = none (ids are >= 0)
};

template <int DIM>
__device__ __forceinline__ int64_t dist2(const Query<DIM>& q, const int4& r) {
    const int dx = q.c[0] - r.x, dy = q.c[1] - r.y;
    int64_t s = (int64_t)dx * dx + (int64_t)dy * dy;
    if (DIM == 3) {
        const int dz = q.c[2] - r.z;
        s += (int64_t)dz * dz;
    }
    return s;
}

// squared distance from q to the box (lo[DIM], hi[DIM]); 0 inside (withinBox)
template <int DIM>
__device__ __forceinline__ int64_t boxd2(const Query<DIM>& q, const int32_t* b) {
    int64_t s = 0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        const int t = max(b[a] - q.c[a], 0) + max(q.c[a] - b[DIM + a], 0);
        s += (int64_t)t * t;
    }
    return s;
}

// Alg. 3 stop test on C's tight box (reading 9): q inside the box with margin m on
// every axis, (m+1)^2 > U.  Every point outside subtree(C) lies outside C's Morton
// cell, which contains the box, so it is at least m+1 away on some axis.
template <int DIM>
__device__ __forceinline__ bool stop_at(const Query<DIM>& q, const int32_t* b, int64_t U) {
    int m = INT_MAX;
#pragma unroll
    for (int a = 0; a < DIM; ++a) m = min(m, min(q.c[a] - b[a], b[DIM + a] - q.c[a]));
    if (m < 0) return false;
    const int64_t mm = (int64_t)m + 1;
    return mm * mm > U;
}

template <int DIM>
__device__ __forceinline__ Node<DIM> load_node(const Node<DIM>* p) {
    Node<DIM> r;
    const int4* s = reinterpret_cast<const int4*>(p);
    int4* d = reinterpret_cast<int4*>(&r);
#pragma unroll
    for (int t = 0; t < (int)(sizeof(Node<DIM>) / 16); ++t) d[t] = __ldg(s + t);
    return r;
}

#ifndef ZD_PW
#define ZD_PW 4
#endif
#ifndef ZD_PW32
#define ZD_PW32 2         // warps per block for 16 < K <= 32
#endif
#ifndef ZD_UNROLL
#define ZD_UNROLL 4
#endif
[[maybe_unused]] constexpr int kUnroll = ZD_UNROLL;   // uniform candidate loop unrolling
template <int K>
struct Pw {
    static constexpr int v = K <= 16 ? ZD_PW : ZD_PW32;   // warps per block (shared memory grows with K)
};
#ifndef ZD_MINB32
#define ZD_MINB32 6       // 2D: min resident blocks per SM for 16 < K <= 32 (the final list spills)
#endif
#ifndef ZD_MINB32_3
#define ZD_MINB32_3 8     // 3D
#endif
#ifndef ZD_MINB
#define ZD_MINB 7         // 2D: min resident blocks per SM for K <= 10 (register budget)
#endif
#ifndef ZD_MINB3
#define ZD_MINB3 8        // 3D (64 registers; with Cap 20 the shared memory fits 8 blocks)
#endif
#ifndef ZD_CH
#define ZD_CH 32
#endif
[[maybe_unused]] constexpr int CH = ZD_CH;                // candidates tested per uniform pass
constexpr int32_t kNoSub = INT32_MIN;    // no subtree pending
#ifndef ZD_STK
#define ZD_STK kMaxDepth
#endif
constexpr int kStk = ZD_STK;             // per-warp stack entries (>= tree height; 64 = key bits + 1)

#ifndef ZD_MINB16
#define ZD_MINB16 5       // 2D: min resident blocks per SM for 10 < K <= 16
#endif
#ifndef ZD_MINB16_3
#define ZD_MINB16_3 6     // 3D
#endif
#ifndef ZD_CAP_MIN
#define ZD_CAP_MIN 22     // 2D
#endif
#ifndef ZD_CAP_MIN3
#define ZD_CAP_MIN3 20    // 3D
#endif
template <int DIM, int K>
struct Cap {   // buffered candidates per lane (overflow compacts per lane: any value > K works)
    static constexpr int cm = DIM == 3 ? ZD_CAP_MIN3 : ZD_CAP_MIN;
    static constexpr int v = (K + 8 > cm) ? K + 8 : cm;
};

// A child reference in traversal form: ref >= 0 internal node; ref < 0 a leaf with
// points [~ref, end).
// A subtree in traversal form with its sorted point range [s, e): ref >= 0 an
// internal node; ref < 0 a contiguous span scanned directly — a leaf, or (query-side
// coarsening) a subtree of at most Coarse<DIM> points, whose points are contiguous too.
#ifndef ZD_COARSE
#define ZD_COARSE 32    // 2D
#endif
#ifndef ZD_COARSE3
#define ZD_COARSE3 96   // 3D (with the fp32 prefilter wide spans are cheap)
#endif
struct Ref {
    int32_t ref, s, e;
};
template <int DIM>
__device__ __forceinline__ Ref child_ref(int32_t c, int32_t s, int32_t e) {
    constexpr int32_t coarse = DIM == 3 ? ZD_COARSE3 : ZD_COARSE;
    return (c < 0 || e - s <= coarse) ? Ref{~s, s, e} : Ref{c, s, e};
}
template <int DIM>
__device__ __forceinline__ Ref left_child(const Node<DIM>& nd, int32_t s) { return child_ref<DIM>(nd.left, s, nd.mid); }
template <int DIM>
__device__ __forceinline__ Ref right_child(const Node<DIM>& nd, int32_t e) { return child_ref<DIM>(nd.right, nd.mid, e); }


#ifndef ZD_PREFETCH_CHILDREN
#define ZD_PREFETCH_CHILDREN 0
#endif
#ifndef ZD_F32FILTER
#define ZD_F32FILTER 1   // 3D: candidate tests in fp32 (exact coordinates), confirmed in int64
#endif
#if !ZD_F32FILTER
#error "the 3D path requires ZD_F32FILTER (fp32 staged candidates)"
#endif
#ifndef ZD_PREFILTER
#define ZD_PREFILTER 1   // drop staged candidates outside the packet box dilated by the span's max bound
#endif
#ifndef ZD_PREGROUPS
#define ZD_PREGROUPS 1   // prefilter boxes per packet (groups of 32 / G Morton-consecutive lanes)
#endif
constexpr int kPG = ZD_PREGROUPS, kPGW = 32 / ZD_PREGROUPS;
#ifndef ZD_SUB
#define ZD_SUB 8         // 2D: candidates per unrolled sub-block of a uniform pass (divides ZD_CH)
#endif
#ifndef ZD_SUB3
#define ZD_SUB3 4        // 3D
#endif
#ifndef ZD_SIGNMASK
#define ZD_SIGNMASK 1    // uniform tests: hit mask from the sign bits of wb - s (3D), U - d2 (2D)
#endif
#ifndef ZD_COOP_OUT
#define ZD_COOP_OUT 1    // stage the packet's output rows in shared memory, write them coalesced
#endif
#ifndef ZD_FIXED_PASS
#define ZD_FIXED_PASS 1  // uniform passes test exactly CH staged slots (masked), self excluded on hits
#endif
#ifndef ZD_PREFILTER2D
#define ZD_PREFILTER2D 0 // the same in 2D (exact int64; measured slightly slower on C2 / 2D Kuzmin)
#endif
// The packed list resolves the bound to 2^-7 only.  A lane whose candidates are far and
// nearly equidistant (relative spread below one bf16 step: an outlier looking at a distant
// dense cluster, a root-based search before its lists settle, the larger bounds of K >=
// 16) then takes EVERY such candidate as a hit instead of the ~K ln N record-breakers:
// measured at 10M points, k = 16 on the Plummer sphere 189 ms instead of 15 ms, root-based
// k = 10 on the 2D Kuzmin disk 9.3 s instead of 19 ms.  So it is used only for K <= 10 in
// leaf-based searches, where the window seed bounds every lane by its 24 Morton
// neighbours first (all five 10M datasets: within the fp32 list's time or 1-7% faster);
// root-based searches with 1 < k <= 10 run on the K = 11 instantiation (fp32 list).
// And even there a constructed input (outliers whose k nearest neighbours are a distant
// dense cluster) hit the same cliff, so the packed list is backed by exact cuts: the
// lane's test bound only decreases (lower_bound_to), and a buffer that stays crowded
// after the cut by that bound is cut at its exact K-th smallest buffered bound, which
// also lowers the test bound (tighten) — the value an fp32 list would hold.
#ifndef ZD_FA_BF16
#define ZD_FA_BF16 1
#endif
#ifndef ZD_FA_BF16_MAXK
#define ZD_FA_BF16_MAXK 10   // (32 reproduces the regression for tests/test_gpu_fullsize.py's time guard)
#endif
template <int K>
constexpr bool kPackedFa = ZD_FA_BF16 && K % 2 == 0 && K <= ZD_FA_BF16_MAXK;
template <int DIM, int K>
struct WarpSh {
    int4 c[DIM == 2 ? 32 : 1];           // 2D: staged candidates (x, y, 0, id)
#if ZD_F32FILTER
    // 3D: the same in fp32 (exact below 2^24), structure of arrays so that one 16-byte
    // load yields one axis of 4 candidates (packed f32x2 tests)
    float fx[32], fy[32], fz[32];
    int32_t fid[32];
#endif
    int32_t p[32];                       // their sorted positions
    float4 pb[2 * kPG];                  // query box of each lane group (lo, hi; 2D: int bits)
    int2 be[Cap<DIM, K>::v][32];              // per-lane buffer (position, fp32 bits of ru(d2)); column = lane
    int4 stk[kStk];                      // (ref, s, e, parent | side << 31): box reloaded on pop
#ifdef ZD_DEBUG
    int32_t dbg_npts, dbg_nint;          // bounds for ZD_DCHECK
#endif
};

template <int DIM, int K>
__device__ __forceinline__ float4 ldf(const WarpSh<DIM, K>& S, int j) {
    return make_float4(S.fx[j], S.fy[j], S.fz[j], __int_as_float(S.fid[j]));
}
template <int DIM, int K>
__device__ __forceinline__ void stf(WarpSh<DIM, K>& S, int j, float4 v) {
    S.fx[j] = v.x; S.fy[j] = v.y; S.fz[j] = v.z; S.fid[j] = __float_as_int(v.w);
}

#ifndef ZD_SEEDW
#define ZD_SEEDW 12      // window seed half-width (all-points queries)
#endif
constexpr int kSeedW = ZD_SEEDW;

// The ascending list fa of the k smallest candidate upper bounds seen so far (only
// fa[K-1], the bound, is ever read).  Even K <= 10: packed bf16 pairs, every value rounded
// UP to bf16 (monotone, so fa[K-1] is the bf16 round-up of the fp32 list's last entry:
// a bound at most 2^-8 looser, never tighter); the median insertion then takes two
// HMNMX2 and one PRMT per pair instead of four FMNMX, in half the registers.
template <int K, bool PACK = kPackedFa<K>>
struct FaList {
    float v[K];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int t = 0; t < K; ++t) v[t] = INFINITY;
    }
    __device__ __forceinline__ float last() const { return v[K - 1]; }
    // insert xf, dropping the largest: every new slot is the median of (v[t-1], xf,
    // v[t]) — all slots independent (depth 2) instead of a K-long compare-exchange
    // chain; xf >= v[K-1] leaves the list unchanged
    __device__ __forceinline__ void insert(float xf) {
#pragma unroll
        for (int t = K - 1; t > 0; --t) v[t] = fmaxf(v[t - 1], fminf(v[t], xf));
        v[0] = fminf(v[0], xf);
    }
};
template <int K>
struct FaList<K, true> {
    uint32_t p[K / 2];   // pair t = (v[2t] in the low half, v[2t+1] in the high half)
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int t = 0; t < K / 2; ++t) p[t] = 0x7f807f80u;   // (+inf, +inf)
    }
    __device__ __forceinline__ float last() const { return __uint_as_float(p[K / 2 - 1] & 0xffff0000u); }
    __device__ __forceinline__ void insert(float xf) {
        // bf16 round-up of xf >= 0 (+inf stays +inf) in both halves
        uint32_t x;
        asm("prmt.b32 %0, %1, 0, 0x3232;" : "=r"(x) : "r"(__float_as_uint(xf) + 0xffffu));
        uint32_t sh[K / 2];   // (v[2t-1], v[2t]) from the old pairs; v[-1] = +0
        sh[0] = p[0] << 16;
#pragma unroll
        for (int t = 1; t < K / 2; ++t) asm("prmt.b32 %0, %1, %2, 0x5432;" : "=r"(sh[t]) : "r"(p[t - 1]), "r"(p[t]));
#pragma unroll
        for (int t = 0; t < K / 2; ++t) {
            uint32_t m;
            asm("min.bf16x2 %0, %1, %2;" : "=r"(m) : "r"(p[t]), "r"(x));
            asm("max.bf16x2 %0, %1, %2;" : "=r"(p[t]) : "r"(sh[t]), "r"(m));
        }
    }
};

template <int DIM, int K>
struct Lane {
    Query<DIM> q;
    FaList<K> fa;
    int64_t U;          // -1 for an idle lane: needs nothing, accepts nothing
    float qf[3];        // 3D fp32 filter: the query in fp32 (exact)
    float wb;           //   and a bound with d2 <= U  =>  fp32 d2 <= wb
    int cnt;
    int32_t wlo;        // window seed: positions [wlo, wlo + 2 * SeedW] were scanned already
#ifdef ZD_KNN_STATS
    bool seed;          // profiling: inside the seed scan
#endif
};

template <int DIM, int K>
__device__ __forceinline__ void set_bound_from(Lane<DIM, K>& L, float f) {
    if (DIM == 3) {
        // 3D: coordinates and their differences are exact in fp32 and the three rounded
        // products/sums make the fp32 d2 at most (1 + 3.0000002 * 2^-24) times the
        // exact one, so d2 <= f implies fp32 d2 <= f * (1 + 2^-21) rounded up
        L.wb = __fmul_ru(f, 1.0f + 0x1p-21f);
    } else {
        L.U = (f == INFINITY) ? INT64_MAX : __float2ll_ru(f);
    }
}
template <int DIM, int K>
__device__ __forceinline__ void set_bound(Lane<DIM, K>& L) {
    set_bound_from<DIM, K>(L, L.fa.last());
}
// the same, never loosening the bound (packed list after tighten(): the test bound may
// already be tighter than the list's bf16 last entry)
template <int DIM, int K>
__device__ __forceinline__ void lower_bound_to(Lane<DIM, K>& L, float f) {
    if (DIM == 3) {
        L.wb = fminf(L.wb, __fmul_ru(f, 1.0f + 0x1p-21f));
    } else {
        const int64_t u = (f == INFINITY) ? INT64_MAX : __float2ll_ru(f);
        L.U = u < L.U ? u : L.U;
    }
}

// fp32 squared distance from q to the box (lo[3], hi[3]): per axis the gap
// max(lo - q, q - hi, 0) (one 3-input max; exact, since lo <= hi and the coordinates
// are exact in fp32), then dx^2, + dy^2, + dz^2 in the candidate test's order.
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float gap_d2(const float (&q)[3], const float* b) {
    const float tx = fmax3(b[0] - q[0], q[0] - b[3], 0.f);
    const float ty = fmax3(b[1] - q[1], q[1] - b[4], 0.f);
    const float tz = fmax3(b[2] - q[2], q[2] - b[5], 0.f);
    return fmaf(tz, tz, fmaf(ty, ty, tx * tx));
}

// (m << 1) | sign bit of x: one funnel shift
__device__ __forceinline__ uint32_t shl_sign(uint32_t m, float x) {
    uint32_t r;
    asm("shf.l.wrap.b32 %0, %1, %2, 1;" : "=r"(r) : "r"(__float_as_uint(x)), "r"(m));
    return r;
}

// Box distance in the lane's test domain: fp32 (3D) or exact int64 (2D).
template <int DIM> struct BoxD { using T = int64_t; };
template <> struct BoxD<3> { using T = float; };
template <int DIM, int K>
__device__ __forceinline__ typename BoxD<DIM>::T box_dist(const Lane<DIM, K>& L, const typename BoxT<DIM>::T* b) {
    if constexpr (DIM == 3) {
        return gap_d2(L.qf, b);
    } else {
        return boxd2<DIM>(L.q, b);
    }
}
template <int DIM, int K>
__device__ __forceinline__ bool within(const Lane<DIM, K>& L, typename BoxD<DIM>::T d) {
    if constexpr (DIM == 3) return d <= L.wb;
    else return d <= L.U;
}

// Is the lane's bound reached by the box (reading 8: visit iff box d2 <= bound)?
// 3D in fp32: per axis max(lo - q, 0) + max(q - hi, 0) is exact, the sum of squares
// errs like a candidate distance, so the test against wb is conservative.
template <int DIM, int K>
__device__ __forceinline__ bool box_need(const Lane<DIM, K>& L, const typename BoxT<DIM>::T* b) {
    if constexpr (DIM == 3) {
        return gap_d2(L.qf, b) <= L.wb;
    } else {
        return boxd2<DIM>(L.q, b) <= L.U;
    }
}

// Alg. 3 stop test (reading 9) on C's box: q inside with margin m on every axis and
// (m+1)^2 > the lane's bound; an idle lane always stops.  3D: m is exact in fp32 and
// (m+1)^2 is rounded down, so the test never stops too early.
template <int DIM, int K>
__device__ __forceinline__ bool lane_stop(const Lane<DIM, K>& L, const typename BoxT<DIM>::T* b) {
    if constexpr (DIM == 3) {
        if (L.wb < 0.f) return true;
        float m = INFINITY;
#pragma unroll
        for (int a = 0; a < 3; ++a) m = fminf(m, fminf(L.qf[a] - b[a], b[3 + a] - L.qf[a]));
        if (m < 0.f) return false;
        const float mm = m + 1.0f;
        return __fmul_rd(mm, mm) > L.fa.last();
    } else {
        return stop_at<DIM>(L.q, b, L.U);
    }
}

// Drop buffered candidates that can no longer qualify: a final neighbour p has
// d2(p) <= the exact k-th smallest d2 seen so far, hence ru(d2(p)) <= fa[K-1].
template <int DIM, int K>
__device__ __forceinline__ void compact(Lane<DIM, K>& L, WarpSh<DIM, K>& S, int lane) {
    // 3D buffers fp32-derived upper bounds ub with d2 <= ub <= d2 (1 + 2^-20): a final
    // neighbour has ub <= D_k (1 + 2^-20) <= fa[K-1] (1 + 2^-20)
    // packed list: the cut comes from the lane's test bound, which only decreases and may
    // be tighter than the list's last entry (tighten): wb >= fK (1 + 2^-21) and U >= fK for
    // the true K-th smallest upper bound fK, so F >= fK (1 + 2^-20) resp. F >= fK as below
    float F;
    if constexpr (kPackedFa<K>) F = DIM == 3 ? __fmul_ru(L.wb, 1.0f + 0x1p-21f) : __ll2float_ru(L.U);
    else F = DIM == 3 ? __fmul_ru(L.fa.last(), 1.0f + 0x1p-20f) : L.fa.last();
    int w = 0;
    for (int e = 0; e < L.cnt; ++e) {
        const int2 v = S.be[e][lane];
        const float f = __int_as_float(v.y);
        S.be[w][lane] = v;
        w += (f <= F) ? 1 : 0;
    }
    L.cnt = w;
}


// Rare path (massive distance ties survive compaction): keep only the exact K best
// buffered candidates by (d2, id).  Entries ranked >= K are marked +inf and dropped
// by the next compaction; the K kept ones all have ru(d2) <= fa[K-1], so later
// compactions keep them.  (Arguments by value: no Lane round trip through memory.)
template <int DIM, int K>
__device__ __noinline__ void mark_exact_losers(const int4* __restrict__ recs, Query<DIM> q, int cnt, WarpSh<DIM, K>& S,
                                               int lane) {
    for (int e = 0; e < cnt; ++e) {
        const int4 ce = __ldg(recs + S.be[e][lane].x);
        const int64_t de = dist2<DIM>(q, ce);
        int rank = 0;
        for (int f = 0; f < cnt; ++f) {
            const int4 cf = __ldg(recs + S.be[f][lane].x);
            const int64_t dv = dist2<DIM>(q, cf);
            rank += (dv < de || (dv == de && cf.w < ce.w)) ? 1 : 0;
        }
        if (rank >= K) S.be[e][lane].y = __float_as_int(INFINITY);
    }
}

// Second-level compaction for a lane whose buffer is still full after compact(): drop
// every entry above the K-th smallest buffered upper bound B (the buffer holds every
// candidate that can still be a final neighbour, so an entry with ub > B — 3D: > B (1 +
// 2^-20), the slack of the fp32-derived bounds — has K strictly closer candidates).
// This is the cut an exact fp32 bound list would make.  The packed bf16 list resolves
// bounds only to 2^-7: a lane that is far from the candidates it is seeing (an
// incoherent packet that was not deferred, a root-based search before its lists settle)
// gets whole spans inside one bf16 step of its bound, and without this cut each overflow
// fell through to mark_exact_losers (O(cnt^2) record loads): C2 root-based k = 10 ran
// 361 ms instead of 10 ms; with it, and with the packed list kept to K <= 10 leaf-based
// searches (FaList), the rare crowded lane costs one O(cnt^2) pass over its own column.
template <int DIM, int K>
__device__ __noinline__ int2 tight_compact(int cnt, WarpSh<DIM, K>& S, int lane) {
    float B = INFINITY;
    for (int e = 0; e < cnt; ++e) {
        const float ue = __int_as_float(S.be[e][lane].y);
        int rank = 0;
        for (int f = 0; f < cnt; ++f) {
            const float uf = __int_as_float(S.be[f][lane].y);
            rank += (uf < ue || (uf == ue && f < e)) ? 1 : 0;
        }
        if (rank == K - 1) B = ue;
    }
    const float F = DIM == 3 ? __fmul_ru(B, 1.0f + 0x1p-20f) : B;
    int w = 0;
    for (int e = 0; e < cnt; ++e) {
        const int2 v = S.be[e][lane];
        S.be[w][lane] = v;
        w += (__int_as_float(v.y) <= F) ? 1 : 0;
    }
    return make_int2(w, __float_as_int(B));   // (new count, the K-th smallest buffered upper bound)
}

// Exact cut of a crowded buffer; with the packed list the K-th smallest buffered bound
// also lowers the lane's test bound (wb / U, which from then on only decrease), so that
// the candidates inside the same bf16 step stop being hits.  It is the value an exact
// fp32 list would hold, so the bound stays as sound as the list's last entry.
template <int DIM, int K>
__device__ __forceinline__ void tighten(Lane<DIM, K>& L, WarpSh<DIM, K>& S, int lane) {
    const int2 r = tight_compact<DIM, K>(L.cnt, S, lane);
    L.cnt = r.x;
    if constexpr (kPackedFa<K>) lower_bound_to<DIM, K>(L, __int_as_float(r.y));
}

// A full buffer must take one more entry: compact by the lane's bound, then by the K-th
// smallest buffered bound, and only on true massive ties rank the survivors exactly.
template <int DIM, int K>
__device__ __forceinline__ void make_room(const int4* __restrict__ recs, Lane<DIM, K>& L, WarpSh<DIM, K>& S, int lane) {
    compact<DIM, K>(L, S, lane);
    if (L.cnt == Cap<DIM, K>::v) {
        tighten<DIM, K>(L, S, lane);
        if (L.cnt == Cap<DIM, K>::v) {   // massive ties: keep only the exact K best
            mark_exact_losers<DIM, K>(recs, L.q, L.cnt, S, lane);
            compact<DIM, K>(L, S, lane);
        }
    }
}

// Every lane scans sorted positions [s, e): up to 32 records at a time are staged
// through shared memory, each lane tests CH of them per uniform pass against its
// bound, then handles its (few) hits.
#ifndef ZD_CROWD
#define ZD_CROWD 3          // packed list: lanes left with more than K + CROWD entries by a uniform compaction take the exact cut
#endif
#ifndef ZD_SLACK
#define ZD_SLACK 2          // uniform compaction when a needing lane has > CAP - SLACK entries (2: measured best of 0-6)
#endif
#ifndef ZD_TRANSPOSE_MAX
#define ZD_TRANSPOSE_MAX 6   // 2D: at most this many needing lanes: lanes = candidates
#endif
#ifndef ZD_TRANSPOSE_MAX3
#define ZD_TRANSPOSE_MAX3 1  // 3D (persistent scheduling: 1 beats 2/3/5 and 0)
#endif
template <int DIM>
struct TMax {
    static constexpr int v = DIM == 3 ? ZD_TRANSPOSE_MAX3 : ZD_TRANSPOSE_MAX;
};
template <int DIM, int K>
__device__ __forceinline__ void scan_span(const int4* __restrict__ recs, int32_t s, int32_t e, bool need,
                                          Lane<DIM, K>& L, WarpSh<DIM, K>& S, int lane) {
    const uint32_t M = __ballot_sync(0xffffffffu, need);
    if (M == 0) return;
    const int w = __popc(M);
    ZD_STAT(ZS_SPANS, 1);
#if ZD_PREFILTER
    // Packet prefilter (uniform mode): a candidate c that some needing lane i accepts
    // is within that lane's bound, bound_i <= bmax (max over the needing lanes), and
    // the distance from c to the packet's query box is at most d2(q_i, c) (per-axis
    // gaps <= |q_i - c|): exact in 2D (int64); in 3D the fp32 box distance uses the
    // same evaluation order on exact per-axis gaps and every rounding is monotone, so
    // it is <= the lane's fp32 d2 <= wb_i.  So dropping c when the box distance exceeds
    // bmax loses nothing; bounds only shrink, so bmax taken here stays valid.
    const bool uni = (DIM == 3 || ZD_PREFILTER2D) && w > TMax<DIM>::v;
    typename BoxD<DIM>::T bmax;
    if constexpr (DIM == 3) bmax = need ? L.wb : -1.0f;
    else bmax = need ? L.U : (int64_t)-1;
    typename BoxD<DIM>::T gm[kPG];   // per lane group (-1: no needing lane in it)
    bool pre = false;
    if (uni) {
#pragma unroll
        for (int o = kPGW >> 1; o > 0; o >>= 1) {
            const typename BoxD<DIM>::T ob = __shfl_xor_sync(0xffffffffu, bmax, o);
            bmax = ob > bmax ? ob : bmax;
        }
        pre = true;
#pragma unroll
        for (int g = 0; g < kPG; ++g) {
            gm[g] = __shfl_sync(0xffffffffu, bmax, g * kPGW);
            if constexpr (DIM == 3) pre = pre && gm[g] != INFINITY;
            else pre = pre && gm[g] != INT64_MAX;
        }
    }
#endif
    for (int32_t b = s; b < e; b += 32) {
        const int n32r = min(32, e - b);
        __syncwarp();
        int4 r = make_int4(0, 0, 0, 0);
        float4 fc = make_float4(0.f, 0.f, 0.f, 0.f);
        bool keep = lane < n32r;
        if (keep) {
#ifdef ZD_DEBUG
            ZD_DCHECK(b >= 0 && b + lane < S.dbg_npts);
#endif
            r = __ldg(recs + b + lane);
#if ZD_F32FILTER
            if (DIM == 3)
                fc = make_float4(__int2float_rn(r.x), __int2float_rn(r.y), __int2float_rn(r.z), __int_as_float(r.w));
#endif
#if ZD_PREFILTER
            if (pre) {
                keep = false;
#pragma unroll
                for (int g = 0; g < kPG; ++g) {
                    const float4 lo = S.pb[2 * g], hi = S.pb[2 * g + 1];
                    if constexpr (DIM == 3) {
                        const float tx = fmax3(lo.x - fc.x, fc.x - hi.x, 0.f);
                        const float ty = fmax3(lo.y - fc.y, fc.y - hi.y, 0.f);
                        const float tz = fmax3(lo.z - fc.z, fc.z - hi.z, 0.f);
                        keep = keep || fmaf(tz, tz, fmaf(ty, ty, tx * tx)) <= gm[g];
                    } else {
                        const int tx = max(__float_as_int(lo.x) - r.x, 0) + max(r.x - __float_as_int(hi.x), 0);
                        const int ty = max(__float_as_int(lo.y) - r.y, 0) + max(r.y - __float_as_int(hi.y), 0);
                        keep = keep || (int64_t)tx * tx + (int64_t)ty * ty <= gm[g];
                    }
                }
            }
#endif
        }
        const uint32_t km = __ballot_sync(0xffffffffu, keep);
        const int n32 = __popc(km);
        if (n32 == 0) continue;
        if (keep) {
            const int slot = __popc(km & ((1u << lane) - 1u));
            if constexpr (DIM == 2) S.c[slot] = r;
            S.p[slot] = b + lane;
#if ZD_F32FILTER
            if (DIM == 3) stf(S, slot, fc);
#endif
        }
        __syncwarp();
#if ZD_CH >= 32
        {   // one pass covers the whole staged chunk (n32 <= 32)
            constexpr int h0 = 0;
            const int cnt = n32;
#else
        for (int h0 = 0; h0 < n32; h0 += CH) {
            const int cnt = min(CH, n32 - h0);
#endif
            // compact (all lanes together) once some needing lane is nearly full; a lane
            // that still fills up while taking hits compacts on its own (take_hit)
            if (__any_sync(0xffffffffu, need && L.cnt > Cap<DIM, K>::v - ZD_SLACK)) {
                ZD_STAT(ZS_COMPACT, 1);
                compact<DIM, K>(L, S, lane);
                // packed list: a buffer still crowded after the cut by the lane's bound holds
                // candidates inside one bf16 step of it (far, nearly equidistant points)
                if constexpr (kPackedFa<K>) {
                    if (L.cnt > K + ZD_CROWD) tighten<DIM, K>(L, S, lane);
                }
            }
            uint32_t hit = 0;
            if (w > TMax<DIM>::v) {
                // every lane tests every candidate against its own bound
#if ZD_FIXED_PASS
                // fixed CH-wide pass (no trip-count checks); slots past cnt hold stale
                // values and are masked off; self is excluded on the hit path
                // in sub-blocks of ZD_SUB (uniform early exit: a short tail costs one
                // sub-block, not a whole pass)
                if constexpr (DIM == 3) {
                    // 4 candidates per step: one 16-byte load per axis, packed f32x2
                    // arithmetic in the same order as the scalar test (dx^2, + dy^2, + dz^2)
                    static_assert(ZD_SUB3 == 4 || ZD_SUB3 == 8, "packed test: 4 or 8 candidates per step");
                    const float wb = L.wb;
                    const float2 qx = make_float2(L.qf[0], L.qf[0]), qy = make_float2(L.qf[1], L.qf[1]),
                                 qz = make_float2(L.qf[2], L.qf[2]);
#if ZD_SIGNMASK
                    // a miss is a negative wb - s (the exact sign of an fp32 difference: the
                    // same decision as s <= wb); each sign bit is shifted into the mask by
                    // one funnel shift, the mask is bit-reversed once per pass
                    const float2 wb2 = make_float2(wb, wb);
                    uint32_t miss = 0;
                    int j0 = 0;
#pragma unroll 1
                    for (; j0 < cnt; j0 += 4) {
                        const float4 X = *reinterpret_cast<const float4*>(&S.fx[h0 + j0]);
                        const float4 Y = *reinterpret_cast<const float4*>(&S.fy[h0 + j0]);
                        const float4 Z = *reinterpret_cast<const float4*>(&S.fz[h0 + j0]);
                        const float2 dx0 = __fadd2_rn(qx, make_float2(-X.x, -X.y)), dx1 = __fadd2_rn(qx, make_float2(-X.z, -X.w));
                        const float2 dy0 = __fadd2_rn(qy, make_float2(-Y.x, -Y.y)), dy1 = __fadd2_rn(qy, make_float2(-Y.z, -Y.w));
                        const float2 dz0 = __fadd2_rn(qz, make_float2(-Z.x, -Z.y)), dz1 = __fadd2_rn(qz, make_float2(-Z.z, -Z.w));
                        const float2 s0 = __ffma2_rn(dz0, dz0, __ffma2_rn(dy0, dy0, __fmul2_rn(dx0, dx0)));
                        const float2 s1 = __ffma2_rn(dz1, dz1, __ffma2_rn(dy1, dy1, __fmul2_rn(dx1, dx1)));
                        const float2 m0 = __fadd2_rn(wb2, make_float2(-s0.x, -s0.y));
                        const float2 m1 = __fadd2_rn(wb2, make_float2(-s1.x, -s1.y));
                        miss = shl_sign(miss, m0.x);
                        miss = shl_sign(miss, m0.y);
                        miss = shl_sign(miss, m1.x);
                        miss = shl_sign(miss, m1.y);
                    }
                    hit = ~(__brev(miss) >> (32 - j0));   // j0 = 4 ceil(cnt / 4) >= 4; candidate j at bit j
#else
#pragma unroll 1
                    for (int j0 = 0; j0 < CH; j0 += ZD_SUB3) {
                        if (j0 >= cnt) break;
#pragma unroll
                        for (int j1 = j0; j1 < j0 + ZD_SUB3; j1 += 4) {
                            const float4 X = *reinterpret_cast<const float4*>(&S.fx[h0 + j1]);
                            const float4 Y = *reinterpret_cast<const float4*>(&S.fy[h0 + j1]);
                            const float4 Z = *reinterpret_cast<const float4*>(&S.fz[h0 + j1]);
                            const float2 dx0 = __fadd2_rn(qx, make_float2(-X.x, -X.y)), dx1 = __fadd2_rn(qx, make_float2(-X.z, -X.w));
                            const float2 dy0 = __fadd2_rn(qy, make_float2(-Y.x, -Y.y)), dy1 = __fadd2_rn(qy, make_float2(-Y.z, -Y.w));
                            const float2 dz0 = __fadd2_rn(qz, make_float2(-Z.x, -Z.y)), dz1 = __fadd2_rn(qz, make_float2(-Z.z, -Z.w));
                            const float2 s0 = __ffma2_rn(dz0, dz0, __ffma2_rn(dy0, dy0, __fmul2_rn(dx0, dx0)));
                            const float2 s1 = __ffma2_rn(dz1, dz1, __ffma2_rn(dy1, dy1, __fmul2_rn(dx1, dx1)));
                            const uint32_t hb = (s0.x <= wb ? 1u : 0u) | (s0.y <= wb ? 2u : 0u) |
                                                (s1.x <= wb ? 4u : 0u) | (s1.y <= wb ? 8u : 0u);
                            hit |= hb << j1;
                        }
                    }
#endif
                } else {
                    const int64_t U = L.U;
#if ZD_SIGNMASK
                    // miss iff U - d2 < 0 (no overflow: 0 <= d2 < 2^63, -1 <= U), the sign
                    // bits funnel-shifted into the mask as in 3D
                    uint32_t miss = 0;
                    int j0 = 0;
#pragma unroll 1
                    for (; j0 < cnt; j0 += ZD_SUB) {
#pragma unroll
                        for (int jj = 0; jj < ZD_SUB; ++jj) {
                            const int4 c = S.c[h0 + j0 + jj];
                            const int64_t m = U - dist2<DIM>(L.q, c);
                            miss = shl_sign(miss, __int_as_float((int)(m >> 32)));
                        }
                    }
                    hit = ~(__brev(miss) >> (32 - j0));   // j0 = ZD_SUB ceil(cnt / ZD_SUB)
#else
#pragma unroll 1
                    for (int j0 = 0; j0 < CH; j0 += ZD_SUB) {
                        if (j0 >= cnt) break;
#pragma unroll
                        for (int jj = 0; jj < ZD_SUB; ++jj) {
                            const int j = j0 + jj;
                            const int4 c = S.c[h0 + j];
                            if (dist2<DIM>(L.q, c) <= U) hit |= 1u << j;
                        }
                    }
#endif
                }
                hit &= cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u);
#else
                if constexpr (DIM == 3) {
                    const float wb = L.wb;
#pragma unroll kUnroll
                    for (int j = 0; j < cnt; ++j) {
                        const float4 c = S.f[h0 + j];
                        const float dx = L.qf[0] - c.x, dy = L.qf[1] - c.y, dz = L.qf[2] - c.z;
                        const float df = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                        const bool h = df <= wb && __float_as_int(c.w) != L.q.id;   // self excluded by id
                        hit |= (h ? 1u : 0u) << j;
                    }
                } else {
                    const int64_t U = L.U;
#pragma unroll kUnroll
                    for (int j = 0; j < cnt; ++j) {
                        const int4 c = S.c[h0 + j];
                        const bool h = dist2<DIM>(L.q, c) <= U && c.w != L.q.id;   // self excluded by id
                        hit |= (h ? 1u : 0u) << j;
                    }
                }
#endif
            } else {
                // few lanes need these candidates: lane j holds candidate j and the warp
                // loops over the needing queries (broadcast by shuffle), one ballot each
                const bool cv = lane < cnt;
                uint32_t m = M;
                if constexpr (DIM == 3) {
                    const float4 c = ldf(S, h0 + (cv ? lane : 0));
                    while (m) {
                        const int i = __ffs(m) - 1;
                        m &= m - 1;
                        const float qx = __shfl_sync(0xffffffffu, L.qf[0], i);
                        const float qy = __shfl_sync(0xffffffffu, L.qf[1], i);
                        const float qz = __shfl_sync(0xffffffffu, L.qf[2], i);
                        const float wbi = __shfl_sync(0xffffffffu, L.wb, i);
                        const int32_t idi = __shfl_sync(0xffffffffu, L.q.id, i);
                        const float dx = qx - c.x, dy = qy - c.y, dz = qz - c.z;
                        const float df = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                        const bool h = cv && df <= wbi && __float_as_int(c.w) != idi;
                        const uint32_t B = __ballot_sync(0xffffffffu, h);
                        if (lane == i) hit = B;
                    }
                } else {
                    const int4 c = S.c[h0 + (cv ? lane : 0)];
                    while (m) {
                        const int i = __ffs(m) - 1;
                        m &= m - 1;
                        Query<DIM> qi;
                        qi.c[0] = __shfl_sync(0xffffffffu, L.q.c[0], i);
                        qi.c[1] = __shfl_sync(0xffffffffu, L.q.c[1], i);
                        qi.c[2] = 0;
                        const int32_t idi = __shfl_sync(0xffffffffu, L.q.id, i);
                        const int64_t Ui = __shfl_sync(0xffffffffu, L.U, i);
                        const bool h = cv && dist2<DIM>(qi, c) <= Ui && c.w != idi;
                        const uint32_t B = __ballot_sync(0xffffffffu, h);
                        if (lane == i) hit = B;
                    }
                }
            }
            {
                // drop the staged slots of the lane's window seed (scanned already): the
                // window is a contiguous range of raw offsets of this chunk, so its staged
                // slots (compacted in order by km) are contiguous too
                const int32_t lo_r = L.wlo - b, hi_r = L.wlo + 2 * kSeedW + 1 - b;   // raw [lo_r, hi_r)
                const bool inw = lo_r < 32 && hi_r > 0;
                if (__any_sync(0xffffffffu, inw) && inw) {
                    const int a = max(lo_r, 0), z = min(hi_r, 32);
                    const int sa = __popc(km & ((1u << a) - 1u));
                    const int sz = __popc(z >= 32 ? km : (km & ((1u << z) - 1u)));
                    hit &= ~((sz >= 32 ? 0xffffffffu : ((1u << sz) - 1u)) & ~((1u << sa) - 1u));
                }
            }
#ifdef ZD_KNN_STATS
            {
                ZD_STAT(ZS_CAND, cnt);
                ZD_STAT(ZS_PASSES, 1);
                ZD_STAT(ZS_NEED_PAIRS, w * cnt);   // pairs if only the needing lanes tested
                ZD_STAT(ZS_RAW, n32r);
                int hc = __popc(hit), hm = hc;
                for (int o = 16; o > 0; o >>= 1) { hm = max(hm, __shfl_xor_sync(0xffffffffu, hm, o)); hc += __shfl_xor_sync(0xffffffffu, hc, o); }
                ZD_STAT(ZS_HITS, hc);
                ZD_STAT(ZS_ROUNDS, hm);
                if (L.seed) { ZD_STAT(ZS_SEED_HITS, hc); ZD_STAT(ZS_SEED_ROUNDS, hm); }
            }
#endif
            while (hit) {
                const int j = h0 + __ffs(hit) - 1;
                hit &= hit - 1;
                float xf;
                bool stale;   // outside the lane's current bound (it shrank since the test)
                if constexpr (DIM == 3) {
                    const float4 c = ldf(S, j);
                    const float dx = L.qf[0] - c.x, dy = L.qf[1] - c.y, dz = L.qf[2] - c.z;
                    const float df = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                    if (__float_as_int(c.w) == L.q.id) continue;   // self (excluded by id, reading 13)
                    stale = df > L.wb;
                    xf = __fmul_ru(df, 1.0f + 0x1p-21f);   // >= the exact d2
                } else {
                    const int4 c = S.c[j];
                    if (c.w == L.q.id) continue;   // self
                    const int64_t d = dist2<DIM>(L.q, c);
                    stale = d > L.U;
                    xf = __ll2float_ru(d);
                }
                if (stale) continue;
#ifdef ZD_KNN_STATS
                atomicAdd(&g_knn_stats[ZS_INS], 1ull);
                if (L.seed) atomicAdd(&g_knn_stats[ZS_SEED_INS], 1ull);
                if (L.cnt == Cap<DIM, K>::v) atomicAdd(&g_knn_stats[ZS_LANE_COMPACT], 1ull);
#endif
                L.fa.insert(xf);
                if constexpr (kPackedFa<K>) lower_bound_to<DIM, K>(L, L.fa.last());
                else set_bound<DIM, K>(L);
                if (L.cnt == Cap<DIM, K>::v) make_room<DIM, K>(recs, L, S, lane);   // rare: per-lane compaction
                ZD_DCHECK((L.cnt < Cap<DIM, K>::v));
                S.be[L.cnt][lane] = make_int2(S.p[j], __float_as_int(xf));
                ++L.cnt;
            }
        }
    }
}

// Seed (Alg. 3's leaf scan, for the whole packet): every lane tests every
// record of [s, e) (the packet's leaves and their neighbours).  Early in a search
// almost every candidate improves the k-best list, so instead of per-hit divergent
// insertions the seed runs two warp-uniform passes:
//   1. fold every candidate's ru(d2) into fa (the branch-free median insertion is a
//      no-op for a value >= fa[K-1]; skipped when no lane would change);
//   2. with the bound of step 1, buffer every candidate within it (the same test as
//      the hit path), so the buffer receives ~k entries and never the whole seed.
// Self (by id, reading 13) and idle lanes take +inf in step 1 and are never buffered.
template <int DIM, int K>
__device__ __forceinline__ void seed_scan(const int4* __restrict__ recs, int32_t s, int32_t e, bool active,
                                          Lane<DIM, K>& L, WarpSh<DIM, K>& S, int lane) {
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
#pragma unroll 1
        for (int32_t b = s; b < e; b += 32) {
            const int n32 = min(32, e - b);
            __syncwarp();
            if (lane < n32) {
                const int4 r = __ldg(recs + b + lane);
                if constexpr (DIM == 3)
                    stf(S, lane, make_float4(__int2float_rn(r.x), __int2float_rn(r.y), __int2float_rn(r.z), __int_as_float(r.w)));
                else
                    S.c[lane] = r;
            }
            __syncwarp();
            if (pass == 0) {
#pragma unroll 1
                for (int j = 0; j < n32; ++j) {
                    float xf;
                    int32_t cid;
                    if constexpr (DIM == 3) {
                        const float4 c = ldf(S, j);
                        const float dx = L.qf[0] - c.x, dy = L.qf[1] - c.y, dz = L.qf[2] - c.z;
                        xf = __fmul_ru(fmaf(dz, dz, fmaf(dy, dy, dx * dx)), 1.0f + 0x1p-21f);   // >= the exact d2
                        cid = __float_as_int(c.w);
                    } else {
                        const int4 c = S.c[j];
                        xf = __ll2float_ru(dist2<DIM>(L.q, c));
                        cid = c.w;
                    }
                    if (!active || cid == L.q.id) xf = INFINITY;
                    if (__any_sync(0xffffffffu, xf < L.fa.last())) L.fa.insert(xf);
                }
            } else {
                const float wb = L.wb;
                const int64_t U = L.U;
#pragma unroll 1
                for (int j = 0; j < n32; ++j) {
                    bool in;
                    float xf;
                    int32_t cid;
                    if constexpr (DIM == 3) {
                        const float4 c = ldf(S, j);
                        const float dx = L.qf[0] - c.x, dy = L.qf[1] - c.y, dz = L.qf[2] - c.z;
                        const float df = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                        in = df <= wb;
                        xf = __fmul_ru(df, 1.0f + 0x1p-21f);
                        cid = __float_as_int(c.w);
                    } else {
                        const int4 c = S.c[j];
                        const int64_t d = dist2<DIM>(L.q, c);
                        in = d <= U;
                        xf = __ll2float_ru(d);
                        cid = c.w;
                    }
                    if (in && cid != L.q.id) {
                        if (L.cnt == Cap<DIM, K>::v) make_room<DIM, K>(recs, L, S, lane);   // rare (ties)
                        S.be[L.cnt][lane] = make_int2(b + j, __float_as_int(xf));
                        ++L.cnt;
                    }
                }
            }
        }
        if (pass == 0) {
            if (active) set_bound<DIM, K>(L);
        }
    }
}

// Window seed (all-points queries): lane i first searches the 2*SeedW sorted positions
// around its own (its Morton neighbours: Alg. 3's leaf seed, widened to a
// fixed window so that every lane does the same amount of uniform work; queries are
// walked in Morton order).  The window's records are staged once per packet in
// shared memory (the idle stack); two passes as in seed_scan: fold every candidate into
// fa, then buffer the candidates within the resulting bound.  The rest of the search
// skips window positions on its hit path (each point is buffered at most once), so the
// traversal covers the whole tree with the window's bound.
template <int DIM, int K>
__device__ __forceinline__ void window_seed(const int4* __restrict__ recs, int32_t n, int32_t p0, bool active,
                                            Lane<DIM, K>& L, WarpSh<DIM, K>& S, int lane) {
    static_assert(32 + 2 * kSeedW <= kStk, "the window is staged in the per-warp stack");
    int4* W = S.stk;
    const int32_t base = p0 - kSeedW;
    __syncwarp();
#pragma unroll
    for (int t = lane; t < 32 + 2 * kSeedW; t += 32) {
        const int32_t pos = base + t;
        int4 v = make_int4(0, 0, 0, -1);   // outside [0, n): never a candidate
        if (pos >= 0 && pos < n) {
            v = __ldg(recs + pos);
            if constexpr (DIM == 3)
                v = make_int4(__float_as_int(__int2float_rn(v.x)), __float_as_int(__int2float_rn(v.y)),
                              __float_as_int(__int2float_rn(v.z)), v.w);
        }
        W[t] = v;
    }
    __syncwarp();
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
        const float wb = L.wb;
        const int64_t U = L.U;
#pragma unroll 4
        for (int j = 0; j <= 2 * kSeedW; ++j) {
            if (j == kSeedW) continue;   // the lane's own position (self)
            const int4 c = W[lane + j];
            float xf;
            bool in;
            if constexpr (DIM == 3) {
                const float dx = L.qf[0] - __int_as_float(c.x), dy = L.qf[1] - __int_as_float(c.y),
                            dz = L.qf[2] - __int_as_float(c.z);
                const float df = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                xf = __fmul_ru(df, 1.0f + 0x1p-21f);   // >= the exact d2
                in = df <= wb;
            } else {
                const int64_t d = dist2<DIM>(L.q, c);
                xf = __ll2float_ru(d);
                in = d <= U;
            }
            const bool valid = active && c.w >= 0;
            if (pass == 0) {
                if (!valid) xf = INFINITY;
                if (__any_sync(0xffffffffu, xf < L.fa.last())) L.fa.insert(xf);
            } else if (valid && in) {
                if (L.cnt == Cap<DIM, K>::v) make_room<DIM, K>(recs, L, S, lane);   // rare (ties)
                S.be[L.cnt][lane] = make_int2(base + lane + j, __float_as_int(xf));
                ++L.cnt;
            }
        }
        if (pass == 0 && active) set_bound<DIM, K>(L);
    }
    __syncwarp();
}

// Scan the spans [s, mid) (lanes with needl) and [mid, e) (lanes with needr; mid == e
// for a single span) minus the already scanned [ps_lo, ps_hi); a lane that needs
// either span tests both.  Two adjacent spans are staged together.
template <int DIM, int K>
__device__ __forceinline__ void scan_leaves(const int4* __restrict__ recs, int32_t s, int32_t mid, int32_t e,
                                            bool needl, bool needr, int32_t ps_lo, int32_t ps_hi, Lane<DIM, K>& L,
                                            WarpSh<DIM, K>& S, int lane) {
    const int32_t a1 = min(e, max(s, ps_lo));   // piece before the scanned span: [s, a1)
    const int32_t b0 = max(s, min(e, ps_hi));   // piece after it: [b0, e)
    // one inlined copy of scan_span for both pieces (code size: the I-cache matters)
#pragma unroll 1
    for (int pc = 0; pc < 2; ++pc) {
        const int32_t x0 = pc ? b0 : s, x1 = pc ? e : a1;
        if (x0 < x1) scan_span<DIM, K>(recs, x0, x1, (needl && x0 < mid) || (needr && x1 > mid), L, S, lane);
    }
}

// Joint Alg. 2 over the subtree `cur` (needed by the lanes with cur_need); the span
// [ps_lo, ps_hi) was scanned already.  Far children wait on a per-warp shared-memory
// stack as (ref, s, e, parent | side << 31); their box is re-read from the parent.
template <int DIM, int K>
__device__ __forceinline__ void joint_down(const int4* __restrict__ recs, const Node<DIM>* __restrict__ nodes, Ref cur,
                                           bool cur_need, int32_t ps_lo, int32_t ps_hi, Lane<DIM, K>& L,
                                           WarpSh<DIM, K>& S, int lane) {
    int sp = 0;
    while (true) {
        bool descend = false, scan = false;
        int32_t ss = cur.s, sm = cur.e, se = cur.e;   // span(s) to scan: [ss, sm) and [sm, se)
        bool sl = cur_need, sr = false;
        if (cur.ref < 0) {
            scan = true;
        } else {
            ZD_STAT(ZS_NODES, 1);
#ifdef ZD_DEBUG
            ZD_DCHECK(cur.ref < S.dbg_nint && cur.s < cur.e && cur.e <= S.dbg_npts);
#endif
            const Node<DIM> nd = load_node<DIM>(nodes + cur.ref);
#if ZD_PREFETCH_CHILDREN
            // warm L1 with both internal children while the boxes are tested
            if (lane == 0 && nd.left >= 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(nodes + nd.left));
            if (lane == 1 && nd.right >= 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(nodes + nd.right));
#endif
            const typename BoxD<DIM>::T dl = box_dist<DIM, K>(L, nd.lbox), dr = box_dist<DIM, K>(L, nd.rbox);
            const bool ln = within<DIM, K>(L, dl), rn = within<DIM, K>(L, dr);
            const bool nl = __any_sync(0xffffffffu, ln), nr = __any_sync(0xffffffffu, rn);
            const Ref lc = left_child<DIM>(nd, cur.s), rc = right_child<DIM>(nd, cur.e);
            if (nl && nr && lc.ref < 0 && rc.ref < 0) {
                // two spans (leaves or small subtrees): adjacent point ranges, one scan
                scan = true;
                sm = nd.mid;
                sl = ln;
                sr = rn;
            } else if (nl && nr) {
                // visit first the child nearer for most lanes (performance only, reading 10)
                const bool lfirst = __popc(__ballot_sync(0xffffffffu, dl <= dr)) >= 16;
                const Ref far = lfirst ? rc : lc;
                __syncwarp();
                ZD_DCHECK(sp < kStk);
                if (lane == 0)
                    S.stk[sp] = make_int4(far.ref, far.s, far.e, (int32_t)((uint32_t)cur.ref | (lfirst ? 0x80000000u : 0u)));
                ++sp;
                cur = lfirst ? lc : rc;
                cur_need = lfirst ? ln : rn;
                descend = true;
            } else if (nl || nr) {
                cur = nl ? lc : rc;
                cur_need = nl ? ln : rn;
                descend = true;
            }
        }
        if (scan) scan_leaves<DIM, K>(recs, ss, sm, se, sl, sr, ps_lo, ps_hi, L, S, lane);
        if (descend) continue;
        // pop the next far child that some lane still needs
        bool found = false;
        __syncwarp();
        while (sp > 0) {
            --sp;
            ZD_STAT(ZS_POPS, 1);
            const int4 e = S.stk[sp];
            typename BoxT<DIM>::T bx[2 * DIM];
            {
                // the far child's box: right box (side bit set) or left box of its parent
                using BT = typename BoxT<DIM>::T;
                const Node<DIM>* pnode = nodes + (e.w & 0x7fffffff);
                const BT* src = (e.w < 0) ? pnode->rbox : pnode->lbox;   // 8-byte aligned
#pragma unroll
                for (int t = 0; t < DIM; ++t) {
                    const int2 v = __ldg(reinterpret_cast<const int2*>(src) + t);
                    bx[2 * t] = *reinterpret_cast<const BT*>(&v.x);
                    bx[2 * t + 1] = *reinterpret_cast<const BT*>(&v.y);
                }
            }
            const bool pn = within<DIM, K>(L, box_dist<DIM, K>(L, bx));
            if (__any_sync(0xffffffffu, pn)) {
                cur = Ref{e.x, e.y, e.z};
                cur_need = pn;
                found = true;
                break;
            }
        }
        if (!found) break;
    }
}

struct PacketArgs {
    const int4* recs;          // tree records (sorted)
    const int32_t* leaf_start;
    const int32_t* leaf_parent;
    const void* nodes;
    const int32_t* node_range;
    const int32_t* split_bit;  // per internal node (in-order)
    const int2* pos_range;     // per internal node: sorted point range [x, y)
    const int4* qrecs;         // queries in Morton order: (x, y, z|0, id or query index)
    const int32_t* qleaf;      // leaf of each query
    int32_t q_lo;              // all-points: first query position (a partition of the sorted points)
    int32_t nq;
    int32_t n_pts;             // tree points (bounds checks)
    const int32_t* d_meta;     // [0] = internal node count (bounds checks)
    int k;
    const int32_t* row_of_id;  // all-points: row of an id (NULL: row = id)
    int32_t* out_idx;
    int64_t* out_d2;
    int32_t* hard_list;        // packets deferred to the second pass (NULL: never defer)
    int32_t* hard_count;       // [0] deferred packets, [1] next packet of the persistent first pass
    int hard_cap;
    int hard_mode;             // 0: packets; 1: second pass over the deferred packets' queries
    int defer_all;             // testing: defer every packet (hard_list must be set)
    int root_based;            // ablation: root-based search instead of leaf-based
};

#ifndef ZD_PERSIST
#define ZD_PERSIST 1     // persistent first pass (needs hard_count[1] zeroed; grid = resident blocks)
#endif
#ifndef ZD_PCHUNK
#define ZD_PCHUNK 1      // packets per fetch of a persistent warp
#endif
#ifndef ZD_INCOHERENT
#define ZD_INCOHERENT 65536.0f  // defer a packet if its extent^2 > this * median bound (retuned under the
                                // persistent first pass: 4096 deferred ~500 packets at C2 / C4b, whose one-query-
                                // per-warp second launch cost more than searching them as packets)
#endif
#ifndef ZD_INCOHERENT16
#define ZD_INCOHERENT16 4096.0f // the same for K >= 16, where the joint search of a spread-out packet costs more
                                // (measured: K2 k = 16 11.9 ms at 4096, 17.7 ms at 16384 and 65536)
#endif


// EXT = false: all-points (queries are the tree's own points; self excluded by id,
// row = row_of_id[id]).  EXT = true: external queries (nothing excluded, row = query
// index carried in the record's w).
// Search the queries at Morton positions [p0, pe) (pe - p0 <= 32) as one packet.
// Returns false (writing nothing) if the packet was deferred to the second pass.
template <int DIM, int K, bool EXT>
__device__ __forceinline__ bool search_packet(const PacketArgs& A, int32_t p0, int32_t pe, int64_t pk, bool can_defer,
                                              WarpSh<DIM, K>& S, int lane) {
    const int32_t p = p0 + lane;
    const bool active = p < pe;
    const int32_t pq = active ? p : p0;
    const int4 r = __ldg(A.qrecs + pq);
#ifdef ZD_KNN_STATS
    const long long t_start = clock64();
#endif
    const Node<DIM>* nodes = static_cast<const Node<DIM>*>(A.nodes);

    Lane<DIM, K> L;
    L.q.c[0] = r.x; L.q.c[1] = r.y; L.q.c[2] = r.z;
    L.q.id = EXT ? -1 : r.w;
    L.fa.init();
    L.U = active ? INT64_MAX : (int64_t)-1;   // an idle lane needs nothing, accepts nothing
    L.qf[0] = __int2float_rn(r.x); L.qf[1] = __int2float_rn(r.y); L.qf[2] = __int2float_rn(r.z);
    L.wb = active ? INFINITY : -1.0f;
    L.cnt = 0;
#if ZD_PREFILTER
    if (DIM == 3 || ZD_PREFILTER2D) {
        // the packet's query box for the prefilter (idle lanes hold a copy of query p0);
        // 3D in fp32 (exact), 2D as int32 bit patterns
        float lo[DIM], hi[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            if constexpr (DIM == 3) {
                lo[a] = L.qf[a];
                hi[a] = L.qf[a];
            }
            int il = L.q.c[a], ih = L.q.c[a];
#pragma unroll
            for (int o = kPGW >> 1; o > 0; o >>= 1) {
                if constexpr (DIM == 3) {
                    lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
                    hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
                } else {
                    il = min(il, __shfl_xor_sync(0xffffffffu, il, o));
                    ih = max(ih, __shfl_xor_sync(0xffffffffu, ih, o));
                }
            }
            if constexpr (DIM == 2) {
                lo[a] = __int_as_float(il);
                hi[a] = __int_as_float(ih);
            }
        }
        if ((lane & (kPGW - 1)) == 0) {
            S.pb[2 * (lane / kPGW)] = make_float4(lo[0], lo[1], DIM == 3 ? lo[DIM - 1] : 0.f, 0.f);
            S.pb[2 * (lane / kPGW) + 1] = make_float4(hi[0], hi[1], DIM == 3 ? hi[DIM - 1] : 0.f, 0.f);
        }
        __syncwarp();
    }
#endif

    int32_t lA, lB;
    if (!EXT) {
        lA = __ldg(A.qleaf + p0);
        lB = __ldg(A.qleaf + pe - 1);
    } else {
        // bit-located leaves of Morton-sorted queries need not be monotone (a skipped
        // bit can route a larger key left): take the packet's min..max, or just the min
        // if that range is wide (any leaf range is a valid seed)
        const int32_t ql = __ldg(A.qleaf + pq);
        lA = ql;
        lB = ql;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lA = min(lA, __shfl_xor_sync(0xffffffffu, lA, o));
            lB = max(lB, __shfl_xor_sync(0xffffffffu, lB, o));
        }
        if (lB - lA > 8) lB = lA;
    }
    // root-based search (ablation): Alg. 2 from the root with an empty list, no
    // leaf seed and no ascent; leaf-based (default): seed with the packet's leaves
#ifndef ZD_SEED_PAD
#define ZD_SEED_PAD 1   // extra Morton-adjacent leaves scanned on each side of the seed
#endif
#ifndef ZD_WSEED
#define ZD_WSEED 1
#endif
    constexpr bool wseed = ZD_WSEED && !EXT;
    int32_t ps_lo = 0, ps_hi = 0;   // sorted range scanned by the packet seed (skipped later)
    L.wlo = INT32_MIN / 2;          // no window: the hit-path window test never fires
#ifdef ZD_KNN_STATS
    L.seed = true;
#endif
    if (A.root_based) {
    } else if (wseed) {
        L.wlo = p - kSeedW;
        window_seed<DIM, K>(A.recs, A.n_pts, p0, active, L, S, lane);
    } else {
        int32_t sA = lA, sB = lB;
        if (ZD_SEED_PAD > 0) {
            const int32_t nleaves = __ldg(A.d_meta) + 1;
            sA = max(0, lA - ZD_SEED_PAD);
            sB = min(nleaves - 1, lB + ZD_SEED_PAD);
        }
        ps_lo = __ldg(A.leaf_start + sA);
        ps_hi = __ldg(A.leaf_start + sB + 1);
        seed_scan<DIM, K>(A.recs, ps_lo, ps_hi, active, L, S, lane);
    }
#ifdef ZD_KNN_STATS
    L.seed = false;
#endif

    if (can_defer && !A.root_based) {
        // A packet whose queries are far apart compared with their neighbour distances
        // (32 Morton-consecutive points straddling a large Morton-cell boundary) would
        // make one warp search several distant regions jointly; it is deferred to a
        // second pass that searches its queries one per warp.
        float ext2 = 0.f;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            int mn = L.q.c[a], mx = L.q.c[a];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            }
            const float e = (float)(mx - mn);
            ext2 = fmaxf(ext2, e * e);
        }
        const bool fin = active && L.fa.last() != INFINITY;
        const int nfin = __popc(__ballot_sync(0xffffffffu, fin));
        const int nact = __popc(__ballot_sync(0xffffffffu, active));
        // median over the active lanes of log2(bound + 1) (bitonic sort across the warp;
        // idle lanes sort last)
        float v = active ? (fin ? __log2f(L.fa.last() + 1.0f) : 1e30f) : INFINITY;
#pragma unroll
        for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
            for (int j = kk >> 1; j > 0; j >>= 1) {
                const float o = __shfl_xor_sync(0xffffffffu, v, j);
                const bool up = (lane & kk) == 0, lower = (lane & j) == 0;
                v = (lower == up) ? fminf(v, o) : fmaxf(v, o);
            }
        }
        const float med = __shfl_sync(0xffffffffu, v, nact >> 1);
        if (A.defer_all || (nfin == nact && ext2 > (K <= 10 ? ZD_INCOHERENT : ZD_INCOHERENT16) * exp2f(med))) {
            int slot = 0;
            if (lane == 0) slot = atomicAdd(A.hard_count, 1);
            slot = __shfl_sync(0xffffffffu, slot, 0);
            if (slot < A.hard_cap) {
                if (lane == 0) A.hard_list[slot] = (int32_t)pk;
                ZD_STAT(ZS_DEFERRED, 1);
                return false;
            }
        }
    }

    // C = the node whose subtree has been searched (-1: the single leaf lA)
    int32_t C = -1, P;
    Ref sub{kNoSub, 0, 0};
    bool sub_need = active;
    if (A.root_based) {
        const int32_t root = __ldg(A.d_meta + 1);   // internal index, or ~0 for a single leaf
        sub = root >= 0 ? child_ref<DIM>(root, 0, A.n_pts) : Ref{~0, 0, A.n_pts};
        P = -1;
    } else if (lA == lB) {
        P = __ldg(A.leaf_parent + lA);
        if (wseed) {   // the window seed did not scan the packet's leaf as a whole
            const int32_t ls = __ldg(A.leaf_start + lA), le = __ldg(A.leaf_start + lA + 1);
            sub = Ref{~ls, ls, le};
        }
    } else {
        // lowest common ancestor of leaves lA < lB = the separator node in [lA, lB)
        // with the highest split bit (the canonical tree is the Cartesian tree of the
        // split bits; two equal bits in a range always have a higher one between them)
        int32_t bb = -2, x = lA;
        for (int32_t i0 = lA; i0 < lB; i0 += 32) {
            const int32_t i = i0 + lane;
            const int32_t v = i < lB ? __ldg(A.split_bit + i) : -2;
            if (v > bb) { bb = v; x = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int32_t ob = __shfl_xor_sync(0xffffffffu, bb, o), ox = __shfl_xor_sync(0xffffffffu, x, o);
            if (ob > bb) { bb = ob; x = ox; }
        }
        C = x;
        P = __ldg(&nodes[x].parent);
        const int2 xr = __ldg(A.pos_range + x);
        sub = child_ref<DIM>(x, xr.x, xr.y);
    }
    while (true) {
        if (sub.ref != kNoSub) joint_down<DIM, K>(A.recs, nodes, sub, sub_need, ps_lo, ps_hi, L, S, lane);
        if (P < 0) break;
        ZD_STAT(ZS_ASCENTS, 1);
#ifdef ZD_DEBUG
        ZD_DCHECK(P < S.dbg_nint);
#endif
        const Node<DIM> nd = load_node<DIM>(nodes + P);
        const bool isl = C >= 0 ? nd.left == C : P == lA;   // leaf l is the left child of node l
        typename BoxT<DIM>::T cb[2 * DIM], sb[2 * DIM];
#pragma unroll
        for (int a = 0; a < 2 * DIM; ++a) {
            cb[a] = isl ? nd.lbox[a] : nd.rbox[a];
            sb[a] = isl ? nd.rbox[a] : nd.lbox[a];
        }
        if (__all_sync(0xffffffffu, lane_stop<DIM, K>(L, cb))) break;
        sub_need = box_need<DIM, K>(L, sb);
        if (__any_sync(0xffffffffu, sub_need)) {
            // the sibling's point range: [mid, end of P) or [start of P, mid)
            const int2 pr = __ldg(A.pos_range + P);
            sub = isl ? right_child<DIM>(nd, pr.y) : left_child<DIM>(nd, pr.x);
        } else {
            sub = Ref{kNoSub, 0, 0};
        }
        C = P;
        P = nd.parent;
    }

    // exact (d2, id) selection of the ~k surviving candidates
    compact<DIM, K>(L, S, lane);
#ifdef ZD_KNN_STATS
    {
        ZD_STAT(ZS_PACKETS, 1);
        int sc = L.cnt, sm = L.cnt;
        for (int o = 16; o > 0; o >>= 1) { sm = max(sm, __shfl_xor_sync(0xffffffffu, sm, o)); sc += __shfl_xor_sync(0xffffffffu, sc, o); }
        ZD_STAT(ZS_SURV, sc);
        ZD_STAT(ZS_SURV_MAX, sm);
        const int nact = __popc(__ballot_sync(0xffffffffu, active));
        ZD_STAT(ZS_QUERIES, nact);
        const long long dt = clock64() - t_start;
        ZD_STAT(ZS_CYCLES, dt);
        ZD_STAT(ZS_HIST0 + min(31, 63 - __clzll(dt | 1)), 1);
        if (lane == 0) atomicMax(&g_knn_stats[ZS_MAXPKT], ((unsigned long long)dt << 24) | (unsigned long long)(p0 >> 5));
    }
#endif
    int32_t row = 0;
    if (active) {
        if (EXT) row = r.w;
        else row = A.row_of_id ? __ldg(A.row_of_id + r.w) : r.w;
    }
    if constexpr (ZD_COOP_OUT && 12 * K <= 8 * Cap<DIM, K>::v) {
        // Exact (d2, id) order of the ~k survivors (reading 14): insertion sort of the
        // lane's buffer column by a comparator that decides from the buffered upper
        // bounds ub (d2 <= ub <= d2 (1 + 2^-20)) whenever they differ by more than that
        // factor, and from the exact int64 d2 and id of both records otherwise.
        const int cnt = L.cnt;
        for (int e = 1; e < cnt; ++e) {
            const int2 v = S.be[e][lane];
            const float xv = __int_as_float(v.y), xv_hi = __fmul_ru(xv, 1.0f + 0x1p-19f);
            int f = e - 1;
            while (f >= 0) {
                const int2 u = S.be[f][lane];
                const float xu = __int_as_float(u.y);
                bool before;   // v before u
                if (xv_hi < xu) before = true;
                else if (__fmul_ru(xu, 1.0f + 0x1p-19f) < xv) before = false;
                else {
                    const int4 cv = __ldg(A.recs + v.x), cu = __ldg(A.recs + u.x);
                    const int64_t dv = dist2<DIM>(L.q, cv), du = dist2<DIM>(L.q, cu);
                    before = dv < du || (dv == du && cv.w < cu.w);
                }
                if (!before) break;
                S.be[f + 1][lane] = u;
                --f;
            }
            S.be[f + 1][lane] = v;
        }
        int32_t pos[K];
#pragma unroll
        for (int t = 0; t < K; ++t) pos[t] = t < cnt ? S.be[t][lane].x : -1;
        // cooperative row writes: the packet's rows are staged in the (now idle) buffer
        // and written element-by-element by consecutive lanes, so one store covers ~3
        // rows instead of 32 scattered ones
        using WS = WarpSh<DIM, K>;
        static_assert(offsetof(WS, be) % 8 == 0, "int64 staging needs 8-byte alignment");
        int64_t* sd = reinterpret_cast<int64_t*>(&S.be[0][0]);
        int32_t* si = reinterpret_cast<int32_t*>(sd + 32 * K);
        __syncwarp();
#pragma unroll
        for (int t = 0; t < K; ++t) {
            int64_t d = INT64_MAX;   // short rows are padded (reading 15)
            int32_t id = -1;
            if (pos[t] >= 0) {
                const int4 c = __ldg(A.recs + pos[t]);
                d = dist2<DIM>(L.q, c);
                id = c.w;
            }
            sd[lane * K + t] = d;
            si[lane * K + t] = id;
        }
        S.p[lane] = active ? row : -1;
        __syncwarp();
#pragma unroll 2
        for (int t = lane; t < 32 * K; t += 32) {
            const int qq = t / K, ss = t - qq * K;
            const int32_t rw = S.p[qq];
            if (rw >= 0 && ss < A.k) {
                A.out_idx[(int64_t)rw * A.k + ss] = si[t];
                A.out_d2[(int64_t)rw * A.k + ss] = sd[t];
            }
        }
    } else {
        KBest<K> best;
        best.init();
        for (int e = 0; e < L.cnt; ++e) {
            const int4 c = __ldg(A.recs + S.be[e][lane].x);
            const int64_t d = dist2<DIM>(L.q, c);
            if (best.accepts(d, c.w)) best.insert(d, c.w);
        }
        if (active) {
            int32_t* oi = A.out_idx + (int64_t)row * A.k;
            int64_t* od = A.out_d2 + (int64_t)row * A.k;
#pragma unroll
            for (int s = 0; s < K; ++s) {
                if (s < A.k) { oi[s] = best.i[s]; od[s] = best.d[s]; }
            }
        }
    }
    return true;
}

template <int DIM, int K, bool EXT>
__global__ void __launch_bounds__(Pw<K>::v * 32, (K <= 11 ? (DIM == 3 ? ZD_MINB3 : ZD_MINB)
                                                    : (K <= 16 ? (DIM == 3 ? ZD_MINB16_3 : ZD_MINB16)
                                                               : (DIM == 3 ? ZD_MINB32_3 : ZD_MINB32)))) knn_packet_kernel(PacketArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSh<DIM, K>* sh = reinterpret_cast<WarpSh<DIM, K>*>(smem_raw);   // Pw<K>::v warps
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSh<DIM, K>& S = sh[wib];
#ifdef ZD_DEBUG
    if (lane == 0) {
        S.dbg_nint = __ldg(A.d_meta);
        S.dbg_npts = A.n_pts;
    }
    __syncwarp();
#endif
    const int64_t gw = (int64_t)blockIdx.x * Pw<K>::v + wib;
    const int64_t qe = (int64_t)A.q_lo + A.nq;   // queries are the positions [q_lo, qe)
    if (!A.hard_mode) {
#if ZD_PERSIST
        // persistent warps: packets are taken in Morton order from a counter, so a warp
        // that finishes early starts the next packet instead of idling until its block's
        // slowest warp is done
        const int64_t npk = ((int64_t)A.nq + 31) / 32;
        (void)gw;
        // a fetch takes ZD_PCHUNK consecutive packets, searched one after the other
        int64_t pk = 0, pk_end = 0;
        while (true) {
            if (pk == pk_end) {
                int64_t c = 0;
                if (lane == 0) c = atomicAdd(reinterpret_cast<unsigned int*>(A.hard_count + 1), 1u);
                c = __shfl_sync(0xffffffffu, c, 0);
                pk = c * ZD_PCHUNK;
                if (pk >= npk) break;
                pk_end = min(pk + ZD_PCHUNK, npk);
            }
            const int64_t p0 = A.q_lo + pk * 32;
            const int32_t pe = (int32_t)(p0 + 32 < qe ? p0 + 32 : qe);
            search_packet<DIM, K, EXT>(A, (int32_t)p0, pe, pk, A.hard_list != nullptr, S, lane);
            ++pk;
        }
#else
        if (gw * 32 >= A.nq) return;   // whole warp exits together
        const int64_t p0 = A.q_lo + gw * 32;
        const int32_t pe = (int32_t)(p0 + 32 < qe ? p0 + 32 : qe);
        search_packet<DIM, K, EXT>(A, (int32_t)p0, pe, gw, A.hard_list != nullptr, S, lane);
#endif
    } else {
        // second pass: the deferred packets' queries, one per warp (grid-stride)
        const int64_t cnt = min(*A.hard_count, A.hard_cap);
        const int64_t total = (int64_t)gridDim.x * Pw<K>::v;
        for (int64_t t = gw; t < cnt * 32; t += total) {
            const int64_t pos = A.q_lo + (int64_t)__ldg(A.hard_list + (t >> 5)) * 32 + (t & 31);
            if (pos < qe) search_packet<DIM, K, EXT>(A, (int32_t)pos, (int32_t)pos + 1, 0, false, S, lane);
        }
    }
}

// Bit-based leaf location: follow the query key's bit at each split.
template <int DIM>
__global__ void __launch_bounds__(256) locate_kernel(const uint64_t* __restrict__ qkeys, int32_t m,
                                                     const Node<DIM>* __restrict__ nodes,
                                                     const int32_t* __restrict__ split_bit,
                                                     const int32_t* __restrict__ meta, int32_t* __restrict__ qleaf) {
    const int32_t i = blockIdx.x * 256 + threadIdx.x;
    if (i >= m) return;
    const uint64_t key = __ldg(qkeys + i);
    int32_t cur = __ldg(meta + 1);   // root: internal index, or ~0 for a single-leaf tree
    int32_t leaf = 0;
    while (cur >= 0) {
        const bool right = (key >> __ldg(split_bit + cur)) & 1u;
        const int32_t child = right ? __ldg(&nodes[cur].right) : __ldg(&nodes[cur].left);
        if (child < 0) { leaf = right ? cur + 1 : cur; break; }   // leaf children of node i: i, i+1
        cur = child;
    }
    qleaf[i] = leaf;
}

PacketArgs packet_args(const KnnArgs& a) {
    PacketArgs A{};
    A.recs = a.recs; A.leaf_start = a.leaf_start; A.leaf_parent = a.leaf_parent;
    A.nodes = a.nodes; A.node_range = a.node_range; A.split_bit = a.split_bit; A.pos_range = a.pos_range;
    A.n_pts = (int32_t)a.n; A.d_meta = a.d_meta;
    A.k = a.k; A.row_of_id = a.row_of_id; A.out_idx = a.out_idx; A.out_d2 = a.out_d2;
    A.hard_list = a.hard_list; A.hard_count = a.hard_count; A.hard_cap = a.hard_cap; A.hard_mode = 0;
    A.defer_all = a.defer_all;
    A.root_based = a.root_based;
    return A;
}

template <int DIM, int K, bool EXT>
void launch_packets(const PacketArgs& A, cudaStream_t st) {
    const int64_t warps = ((int64_t)A.nq + 31) / 32;
    int grid = (int)((warps + Pw<K>::v - 1) / Pw<K>::v);
    if (grid <= 0) return;
    const size_t smem = sizeof(WarpSh<DIM, K>) * Pw<K>::v;
    static PerDeviceOnce attr;   // per template instance and device (concurrent zd_knn calls)
    static int resident[64];     // per device: SMs x resident blocks of this instance
    attr.run([&](int dev) {
        cudaFuncSetAttribute(knn_packet_kernel<DIM, K, EXT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int sms = 148, per = 1;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, knn_packet_kernel<DIM, K, EXT>, Pw<K>::v * 32, smem);
        if (dev >= 0 && dev < 64) resident[dev] = sms * (per > 0 ? per : 1);
    });
#if ZD_PERSIST
    {
        int dev = 0;
        cudaGetDevice(&dev);
        const int r = (dev >= 0 && dev < 64 && resident[dev] > 0) ? resident[dev] : 148 * 8;
        grid = std::min(grid, r);
    }
#endif
    count_launch(1);
    knn_packet_kernel<DIM, K, EXT><<<grid, Pw<K>::v * 32, smem, st>>>(A);
    if (A.hard_list) {
        PacketArgs H = A;
        H.hard_mode = 1;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        count_launch(1);
        knn_packet_kernel<DIM, K, EXT><<<sms * 4, Pw<K>::v * 32, smem, st>>>(H);
    }
}

#define ZD_K_CASES(X) X(1) X(4) X(8) X(10) X(16) X(32)

template <int DIM, bool EXT>
void dispatch(const PacketArgs& A, cudaStream_t st) {
    // root-based searches (ablation) keep the fp32 bound list: K = 1, else the odd K = 11
    if (A.root_based && A.k > 1 && A.k <= 11) { launch_packets<DIM, 11, EXT>(A, st); return; }
#define X(KK) if (A.k <= KK) { launch_packets<DIM, KK, EXT>(A, st); return; }
    ZD_K_CASES(X)
#undef X
}

}  // namespace

int knn_stats(unsigned long long* out, int n, int reset) {
#ifdef ZD_KNN_STATS
    if (n > ZD_NSTATS) n = ZD_NSTATS;
    if (cudaMemcpyFromSymbol(out, g_knn_stats, n * sizeof(unsigned long long)) != cudaSuccess) return -1;
    if (reset) {
        unsigned long long z[ZD_NSTATS] = {};
        cudaMemcpyToSymbol(g_knn_stats, z, sizeof(z));
    }
    return n;
#else
    (void)out; (void)n; (void)reset;
    return -1;
#endif
}

void knn_all(const KnnArgs& a, cudaStream_t st) {
    PacketArgs A = packet_args(a);
    A.qrecs = a.recs;
    A.qleaf = a.pt_leaf;
    A.q_lo = (int32_t)a.q_lo;
    A.nq = (int32_t)(a.q_hi - a.q_lo);
    if (A.nq <= 0) return;
    if (a.warp || a.k > kPacketKMax) { knn_warp(a, a.recs + a.q_lo, a.pt_leaf + a.q_lo, A.nq, false, st); return; }
    if (a.dim == 2) dispatch<2, false>(A, st); else dispatch<3, false>(A, st);
}

void knn_queries(const KnnArgs& a, const uint64_t* qkeys, const int4* qrecs, int32_t* qleaf, int64_t m,
                 cudaStream_t st) {
    if (m <= 0) return;
    const int grid = (int)((m + 255) / 256);
    count_launch(1);
    if (a.dim == 2)
        locate_kernel<2><<<grid, 256, 0, st>>>(qkeys, (int32_t)m, (const Node<2>*)a.nodes, a.split_bit, a.d_meta, qleaf);
    else
        locate_kernel<3><<<grid, 256, 0, st>>>(qkeys, (int32_t)m, (const Node<3>*)a.nodes, a.split_bit, a.d_meta, qleaf);
    PacketArgs A = packet_args(a);
    A.qrecs = qrecs;
    A.qleaf = qleaf;
    A.q_lo = 0;
    A.nq = (int32_t)m;
    if (a.warp || a.k > kPacketKMax) { knn_warp(a, qrecs, qleaf, m, true, st); return; }
    if (a.dim == 2) dispatch<2, true>(A, st); else dispatch<3, true>(A, st);
}

}  // namespace zd
