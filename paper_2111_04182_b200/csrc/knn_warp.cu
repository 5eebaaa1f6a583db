// knn_warp.cu — large-k exact k-NN (k up to ZD_K_MAX): one warp per query.
//
// PAPER.md: Alg. 3 searchUp calling Alg. 2 searchDown,
// leaf-based or root-based; the k-best container for large k is a
// priority queue in the paper ("vector for small k, heap for large k"); here
// it is a warp-cooperative buffer with radix selection.
//
// The packet kernel (knn.cu) keeps a k-long list per lane in registers, which stops
// paying beyond k = 32 (register pressure).  Here one warp owns ONE query
// and its traversal is warp-uniform (every lane computes the same node tests, so
// nothing diverges); the 32 lanes share the leaf scans (lane = candidate) and the
// k-best bookkeeping:
//   buf    (exact d2, sorted position) of every candidate with d2 <= T when seen,
//          in shared memory, appended by ballot + prefix rank;
//   T      a bound on the exact k-th smallest d2 seen so far (INT64_MAX until k
//          candidates are buffered); T never grows, and pruning (reading 8), the stop
//          test (reading 9) and buffering by "d2 <= T" lose nothing;
//   select when the buffer would overflow: radix-select (4 x 8 bits) the k-th smallest
//          key ru(d2) (fp32 rounded up, monotone in d2), T = that key as an integer
//          (>= the exact k-th smallest d2), keep the entries with d2 <= T.
// At the end the survivors are ranked exactly by (d2, id) (reading 14) and the first
// k written; short rows are padded with (-1, INT64_MAX) (reading 15).
#include <climits>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace zd {
namespace {

constexpr int KW_CAP = 2 * 128 + 64;   // buffered candidates per query (>= ZD_K_MAX + 32)
constexpr int KW_WARPS = 4;            // warps (queries) per block
constexpr int KW_STK = kMaxDepth;      // DFS stack: at most one far child per tree level
#ifndef ZD_KW_COARSE
#define ZD_KW_COARSE 128               // subtrees of <= this many points are scanned as one span (32-wide chunks)
#endif
#ifndef ZD_KW_MINB
#define ZD_KW_MINB 8
#endif

struct KwSh {
    int64_t d2[KW_CAP];
    int32_t pos[KW_CAP];   // sorted positions; replaced by ids for the final ranking
    uint32_t hist[256];
    int4 stk[KW_STK];      // (ref, s, e, box d2 rounded down, fp32 bits)
};

struct KwArgs {
    const int4* recs;
    const int32_t* leaf_start;
    const int32_t* leaf_parent;
    const void* nodes;
    const int2* pos_range;
    const int32_t* d_meta;     // [0] internal node count, [1] root ref
    const int4* qrecs;         // queries in Morton order (x, y, z|0, id or query index)
    const int32_t* qleaf;      // leaf of each query
    int32_t nq, n_pts, k;
    const int32_t* row_of_id;
    int32_t* out_idx;
    int64_t* out_d2;
    int ext, root_based;
    unsigned int* next;        // persistent warps: next query (zeroed by the caller)
};

struct Sub {
    int32_t ref, s, e;   // ref >= 0 internal node; ref < 0 a span [s, e) scanned directly
};
__device__ __forceinline__ Sub sub_ref(int32_t c, int32_t s, int32_t e) {
    return (c < 0 || e - s <= ZD_KW_COARSE) ? Sub{~s, s, e} : Sub{c, s, e};
}

template <int DIM>
struct KwQuery {
    int c[3];
    int32_t id;   // excluded id (-1: none)
};

template <int DIM>
__device__ __forceinline__ int64_t kw_d2(const KwQuery<DIM>& q, const int4& r) {
    const int dx = q.c[0] - r.x, dy = q.c[1] - r.y;
    int64_t s = (int64_t)dx * dx + (int64_t)dy * dy;
    if (DIM == 3) {
        const int dz = q.c[2] - r.z;
        s += (int64_t)dz * dz;
    }
    return s;
}

// exact squared distance from q to a box (lo[DIM], hi[DIM]) stored as int32 (2D) or
// exact-integer fp32 (3D); 0 inside (withinBox)
template <int DIM>
__device__ __forceinline__ int64_t kw_boxd2(const KwQuery<DIM>& q, const typename BoxT<DIM>::T* b) {
    int64_t s = 0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        const int lo = (int)b[a], hi = (int)b[DIM + a];
        const int t = max(lo - q.c[a], 0) + max(q.c[a] - hi, 0);
        s += (int64_t)t * t;
    }
    return s;
}

// Alg. 3 stop test on C's box (reading 9): q inside with margin m on every axis and
// (m+1)^2 > T
template <int DIM>
__device__ __forceinline__ bool kw_stop(const KwQuery<DIM>& q, const typename BoxT<DIM>::T* b, int64_t T) {
    int m = INT_MAX;
#pragma unroll
    for (int a = 0; a < DIM; ++a) m = min(m, min(q.c[a] - (int)b[a], (int)b[DIM + a] - q.c[a]));
    if (m < 0) return false;
    const int64_t mm = (int64_t)m + 1;
    return mm * mm > T;
}

__device__ __forceinline__ uint32_t kw_key(int64_t d2) { return __float_as_uint(__ll2float_ru(d2)); }

struct KwState {
    int64_t T;
    int cnt;
    int lim;     // re-select once cnt reaches this (first at k: the first finite bound)
    float tf;    // ru(T) (INFINITY while T is INT64_MAX)
    float wb;    // 3D fp32 box tests: exact box d2 <= T  =>  fp32 box d2 <= wb
};

__device__ __forceinline__ void kw_set_T(KwState& st, int64_t T) {
    st.T = T;
    st.tf = __ll2float_ru(T);
    // the fp32 sum of three exact squares is at most (1 + 3.0000002 * 2^-24) times the
    // exact one (as in knn.cu set_bound), so exact <= T implies fp32 <= wb
    st.wb = __fmul_ru(st.tf, 1.0f + 0x1p-21f);
}

// Box distance in the test domain: fp32 in 3D (exact per-axis gaps), exact int64 in 2D.
template <int DIM> struct KwBD { using T = int64_t; };
template <> struct KwBD<3> { using T = float; };
template <int DIM>
__device__ __forceinline__ typename KwBD<DIM>::T kw_bd(const KwQuery<DIM>& q, const float* qf,
                                                        const typename BoxT<DIM>::T* b) {
    if constexpr (DIM == 3) {
        float df = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float t = fmaxf(b[a] - qf[a], 0.f) + fmaxf(qf[a] - b[3 + a], 0.f);
            df = fmaf(t, t, df);
        }
        return df;
    } else {
        return kw_boxd2<DIM>(q, b);
    }
}
template <int DIM>
__device__ __forceinline__ bool kw_within(const KwState& st, typename KwBD<DIM>::T v) {
    if constexpr (DIM == 3) return v <= st.wb;
    else return v <= st.T;
}
// stack form of a box distance (fp32 bits): 3D the fp32 value itself; 2D rounded down
template <int DIM>
__device__ __forceinline__ int kw_bd_bits(typename KwBD<DIM>::T v) {
    if constexpr (DIM == 3) return __float_as_int(v);
    else return __float_as_int(__ll2float_rd(v));
}
template <int DIM>
__device__ __forceinline__ bool kw_bits_within(const KwState& st, int bits) {
    if constexpr (DIM == 3) return __int_as_float(bits) <= st.wb;
    else return (int64_t)__int_as_float(bits) <= st.T;   // value <= exact box d2
}
// Alg. 3 stop test (reading 9) on C's box: 3D in fp32 — m exact, (m+1)^2 rounded down
// against ru(T), so it never stops too early; 2D exact.
template <int DIM>
__device__ __forceinline__ bool kw_stop_t(const KwQuery<DIM>& q, const float* qf, const typename BoxT<DIM>::T* b,
                                          const KwState& st) {
    if constexpr (DIM == 3) {
        float m = INFINITY;
#pragma unroll
        for (int a = 0; a < 3; ++a) m = fminf(m, fminf(qf[a] - b[a], b[3 + a] - qf[a]));
        if (m < 0.f) return false;
        const float mm = m + 1.0f;
        return __fmul_rd(mm, mm) > st.tf;
    } else {
        return kw_stop<DIM>(q, b, st.T);
    }
}

// keep the buffered entries with d2 <= T (stable, in place: write index <= read index)
__device__ __forceinline__ void kw_compact(KwSh& S, KwState& st, int lane) {
    int w = 0;
    for (int base = 0; base < st.cnt; base += 32) {
        const int e = base + lane;
        const bool v = e < st.cnt;
        const int64_t d = v ? S.d2[e] : 0;
        const int32_t p = v ? S.pos[e] : 0;
        const bool keep = v && d <= st.T;
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) {
            const int slot = w + __popc(m & ((1u << lane) - 1u));
            S.d2[slot] = d;
            S.pos[slot] = p;
        }
        w += __popc(m);
        __syncwarp();
    }
    st.cnt = w;
}

// T = the k-th smallest ru(d2) among the buffer (as an integer, >= the exact k-th
// smallest d2); requires cnt >= k.  Radix selection over the fp32 key bits (non-
// negative floats order like their bit patterns), 8 bits per pass.
__device__ __forceinline__ void kw_select(KwSh& S, KwState& st, int k, int lane) {
    uint32_t prefix = 0, mask = 0;
    int kk = k;   // 1-based rank still to find among the entries matching the prefix
#pragma unroll 1
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = lane; i < 256; i += 32) S.hist[i] = 0;
        __syncwarp();
        for (int e = lane; e < st.cnt; e += 32) {
            const uint32_t key = kw_key(S.d2[e]);
            if ((key & mask) == prefix) atomicAdd(&S.hist[(key >> shift) & 255u], 1u);
        }
        __syncwarp();
        uint32_t h[8];
        uint32_t loc = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            h[j] = S.hist[lane * 8 + j];
            loc += h[j];
        }
        uint32_t incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t excl = incl - loc;
        const bool mine = excl < (uint32_t)kk && (uint32_t)kk <= incl;
        int bin = 0;
        uint32_t below = excl;
        if (mine) {
            uint32_t run = excl;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (run + h[j] >= (uint32_t)kk) { bin = lane * 8 + j; below = run; break; }
                run += h[j];
            }
        }
        const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
        bin = __shfl_sync(0xffffffffu, bin, src);
        below = __shfl_sync(0xffffffffu, below, src);
        prefix |= (uint32_t)bin << shift;
        mask |= 255u << shift;
        kk -= (int)below;
        __syncwarp();
    }
    // an fp32 value >= 2^24 is an integer, and below 2^24 ru(d2) == d2: exact conversion
    const int64_t T = (int64_t)__uint_as_float(prefix);
    if (T < st.T) kw_set_T(st, T);
}

// Massive ties (rare): keep exactly the k best buffered entries by (d2, id).
__device__ __noinline__ void kw_keep_exact(const int4* __restrict__ recs, KwSh& S, KwState& st, int k, int lane) {
    const int c = st.cnt;
    for (int base = 0; base < c; base += 32) {
        const int e = base + lane;
        int rank = INT_MAX;
        if (e < c) {
            const int64_t de = S.d2[e];
            const int32_t ie = __ldg(recs + S.pos[e]).w;
            rank = 0;
            for (int f = 0; f < c; ++f) {
                const int64_t df = S.d2[f];
                if (df < de || (df == de && __ldg(recs + S.pos[f]).w < ie)) ++rank;
            }
        }
        __syncwarp();
        if (e < c && rank >= k) S.d2[e] = INT64_MAX;   // dropped by the compaction below
        __syncwarp();
    }
    kw_compact(S, st, lane);
}

// Sort buf[0, c) ascending by (d2, id) (pos[] holds ids here; ids are distinct):
// bitonic network over the next power of two >= c, padded with (INT64_MAX, INT_MAX).
constexpr int kSortMax = 256;   // <= KW_CAP
__device__ __forceinline__ void kw_sort(KwSh& S, int c, int lane) {
    int P = 32;
    while (P < c) P <<= 1;
    ZD_DCHECK(P <= KW_CAP);
    for (int e = c + lane; e < P; e += 32) { S.d2[e] = INT64_MAX; S.pos[e] = INT_MAX; }
    __syncwarp();
#pragma unroll 1
    for (int size = 2; size <= P; size <<= 1) {
#pragma unroll 1
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = lane; t < (P >> 1); t += 32) {
                const int i = 2 * stride * (t / stride) + (t % stride), j = i + stride;
                const bool asc = (i & size) == 0;
                const int64_t di = S.d2[i], dj = S.d2[j];
                const int32_t pi = S.pos[i], pj = S.pos[j];
                const bool gt = di > dj || (di == dj && pi > pj);
                if (gt == asc) {
                    S.d2[i] = dj; S.d2[j] = di;
                    S.pos[i] = pj; S.pos[j] = pi;
                }
            }
            __syncwarp();
        }
    }
}

// Scan sorted positions [s, e): lane = candidate, hits appended to the buffer.
template <int DIM>
__device__ __forceinline__ void kw_scan(const int4* __restrict__ recs, int32_t s, int32_t e, const KwQuery<DIM>& q,
                                        KwSh& S, KwState& st, int k, int lane) {
    for (int32_t b = s; b < e; b += 32) {
        const int32_t p = b + lane;
        int64_t d = INT64_MAX;
        bool hit = false;
        if (p < e) {
            const int4 r = __ldg(recs + p);
            d = kw_d2<DIM>(q, r);
            hit = d <= st.T && r.w != q.id;
        }
        uint32_t m = __ballot_sync(0xffffffffu, hit);
        if (m == 0) continue;
        if (st.cnt + __popc(m) > KW_CAP) {
            kw_select(S, st, k, lane);
            kw_compact(S, st, lane);
            if (st.cnt + 32 > KW_CAP) kw_keep_exact(recs, S, st, k, lane);
            hit = hit && d <= st.T;
            m = __ballot_sync(0xffffffffu, hit);
        }
        if (hit) {
            const int slot = st.cnt + __popc(m & ((1u << lane) - 1u));
            ZD_DCHECK(slot < KW_CAP && p >= 0);
            S.d2[slot] = d;
            S.pos[slot] = p;
        }
        st.cnt += __popc(m);
        __syncwarp();
        if (st.cnt >= st.lim) {
            // tighten T: at k buffered candidates (the first finite bound), then each
            // time the buffer has grown by max(k, 32) since the last selection
            kw_select(S, st, k, lane);
            kw_compact(S, st, lane);
            st.lim = min(st.cnt + max(k, 32), KW_CAP);
        }
    }
}

template <int DIM>
__device__ __forceinline__ Node<DIM> kw_load_node(const Node<DIM>* p) {
    Node<DIM> r;
    const int4* s = reinterpret_cast<const int4*>(p);
    int4* d = reinterpret_cast<int4*>(&r);
#pragma unroll
    for (int t = 0; t < (int)(sizeof(Node<DIM>) / 16); ++t) d[t] = __ldg(s + t);
    return r;
}

// Alg. 2 searchDown of `cur` for one query (warp-uniform DFS; nearer child first,
// reading 10; the far child waits on the stack with its box distance rounded down).
template <int DIM>
__device__ __forceinline__ void kw_down(const KwArgs& A, const Node<DIM>* __restrict__ nodes, Sub cur,
                                        const KwQuery<DIM>& q, const float* qf, KwSh& S, KwState& st, int lane) {
    int sp = 0;
    while (true) {
        bool descend = false;
        if (cur.ref < 0) {
            kw_scan<DIM>(A.recs, cur.s, cur.e, q, S, st, A.k, lane);
        } else {
            const Node<DIM> nd = kw_load_node<DIM>(nodes + cur.ref);
            const typename KwBD<DIM>::T dl = kw_bd<DIM>(q, qf, nd.lbox), dr = kw_bd<DIM>(q, qf, nd.rbox);
            const bool ln = kw_within<DIM>(st, dl), rn = kw_within<DIM>(st, dr);
            const Sub lc = sub_ref(nd.left, cur.s, nd.mid), rc = sub_ref(nd.right, nd.mid, cur.e);
            if (ln && rn) {
                const bool lfirst = dl <= dr;
                const Sub far = lfirst ? rc : lc;
                const int fb = kw_bd_bits<DIM>(lfirst ? dr : dl);
                ZD_DCHECK(sp < KW_STK);
                __syncwarp();
                if (lane == 0) S.stk[sp] = make_int4(far.ref, far.s, far.e, fb);
                ++sp;
                cur = lfirst ? lc : rc;
                descend = true;
            } else if (ln || rn) {
                cur = ln ? lc : rc;
                descend = true;
            }
        }
        if (descend) continue;
        bool found = false;
        __syncwarp();
        while (sp > 0) {
            const int4 e = S.stk[--sp];
            if (kw_bits_within<DIM>(st, e.w)) {
                cur = Sub{e.x, e.y, e.z};
                found = true;
                break;
            }
        }
        if (!found) break;
    }
}

// one query (Morton position qi) searched by the whole warp
template <int DIM>
__device__ __forceinline__ void kw_query(const KwArgs& A, int64_t qi, KwSh& S, int lane) {
    const Node<DIM>* nodes = static_cast<const Node<DIM>*>(A.nodes);
    const int4 r = __ldg(A.qrecs + qi);
    KwQuery<DIM> q;
    q.c[0] = r.x; q.c[1] = r.y; q.c[2] = r.z;
    q.id = A.ext ? -1 : r.w;
    KwState st{INT64_MAX, 0, A.k, INFINITY, INFINITY};
    const float qf[3] = {(float)r.x, (float)r.y, (float)r.z};   // exact (3D: < 2^21)

    if (A.root_based) {
        // Alg. 2 from the root with an empty list, no ascent
        const int32_t root = __ldg(A.d_meta + 1);
        kw_down<DIM>(A, nodes, root >= 0 ? sub_ref(root, 0, A.n_pts) : Sub{~0, 0, A.n_pts}, q, qf, S, st, lane);
    } else {
        // Alg. 3: scan the query's leaf, then ascend; at each ancestor stop if the ball
        // lies inside C's box, else search the sibling subtree
        const int32_t l = __ldg(A.qleaf + qi);
        ZD_DCHECK(l >= 0 && l <= __ldg(A.d_meta));
        kw_scan<DIM>(A.recs, __ldg(A.leaf_start + l), __ldg(A.leaf_start + l + 1), q, S, st, A.k, lane);
        int32_t C = -1, P = __ldg(A.leaf_parent + l);
        while (P >= 0) {
            const Node<DIM> nd = kw_load_node<DIM>(nodes + P);
            const bool isl = C >= 0 ? nd.left == C : P == l;   // leaf l is the left child of node l
            const typename BoxT<DIM>::T* cb = isl ? nd.lbox : nd.rbox;
            const typename BoxT<DIM>::T* sb = isl ? nd.rbox : nd.lbox;
            if (kw_stop_t<DIM>(q, qf, cb, st)) break;
            if (kw_within<DIM>(st, kw_bd<DIM>(q, qf, sb))) {
                const int2 pr = __ldg(A.pos_range + P);
                kw_down<DIM>(A, nodes, isl ? sub_ref(nd.right, nd.mid, pr.y) : sub_ref(nd.left, pr.x, nd.mid), q, qf,
                             S, st, lane);
            }
            C = P;
            P = nd.parent;
        }
    }

    // final: trim to ~k, then rank exactly by (d2, id)
    if (st.cnt > A.k) {
        kw_select(S, st, A.k, lane);
        kw_compact(S, st, lane);
    }
    if (st.cnt > kSortMax) kw_keep_exact(A.recs, S, st, A.k, lane);   // massive ties: exactly k left
    const int c = st.cnt;
    for (int e = lane; e < c; e += 32) S.pos[e] = __ldg(A.recs + S.pos[e]).w;   // positions -> ids
    int64_t row;
    if (A.ext) row = r.w;
    else row = A.row_of_id ? __ldg(A.row_of_id + r.w) : r.w;
    int32_t* oi = A.out_idx + row * A.k;
    int64_t* od = A.out_d2 + row * A.k;
    if (c <= 32) {
        // one survivor per lane: its rank by counting (c steps)
        __syncwarp();
        if (lane < c) {
            const int64_t de = S.d2[lane];
            const int32_t ie = S.pos[lane];
            int rank = 0;
            for (int f = 0; f < c; ++f) {
                const int64_t df = S.d2[f];
                rank += (df < de || (df == de && S.pos[f] < ie)) ? 1 : 0;
            }
            if (rank < A.k) { oi[rank] = ie; od[rank] = de; }
        }
        for (int t = c + lane; t < A.k; t += 32) { oi[t] = -1; od[t] = INT64_MAX; }
    } else {
        kw_sort(S, c, lane);
        for (int t = lane; t < A.k; t += 32) {
            const bool v = t < c;
            oi[t] = v ? S.pos[t] : -1;
            od[t] = v ? S.d2[t] : INT64_MAX;
        }
    }
}

// Persistent warps: each takes the next query in Morton order from a counter (a warp
// that finishes early starts another query instead of idling until its block is done).
template <int DIM>
__global__ void __launch_bounds__(KW_WARPS * 32, ZD_KW_MINB) knn_warp_kernel(KwArgs A) {
    __shared__ KwSh sh[KW_WARPS];
    const int lane = threadIdx.x & 31;
    KwSh& S = sh[threadIdx.x >> 5];
    while (true) {
        int64_t qi = 0;
        if (lane == 0) qi = atomicAdd(A.next, 1u);
        qi = __shfl_sync(0xffffffffu, qi, 0);
        if (qi >= A.nq) break;   // whole warp
        kw_query<DIM>(A, qi, S, lane);
        __syncwarp();
    }
}

}  // namespace

void knn_warp(const KnnArgs& a, const int4* qrecs, const int32_t* qleaf, int64_t nq, bool ext, cudaStream_t st) {
    if (nq <= 0) return;
    KwArgs A{};
    A.recs = a.recs; A.leaf_start = a.leaf_start; A.leaf_parent = a.leaf_parent; A.nodes = a.nodes;
    A.pos_range = a.pos_range; A.d_meta = a.d_meta; A.qrecs = qrecs; A.qleaf = qleaf;
    A.nq = (int32_t)nq; A.n_pts = (int32_t)a.n; A.k = a.k; A.row_of_id = ext ? nullptr : a.row_of_id;
    A.out_idx = a.out_idx; A.out_d2 = a.out_d2; A.ext = ext ? 1 : 0; A.root_based = a.root_based;
    A.next = reinterpret_cast<unsigned int*>(a.hard_count + 1);   // zeroed by zd_knn
    int grid = (int)((nq + KW_WARPS - 1) / KW_WARPS);
    static PerDeviceOnce occ;
    static int resident[2][64];   // per dimension and device: SMs x resident blocks
    occ.run([&](int dev) {
        int sms = 148, p2 = 1, p3 = 1;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2, knn_warp_kernel<2>, KW_WARPS * 32, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p3, knn_warp_kernel<3>, KW_WARPS * 32, 0);
        if (dev >= 0 && dev < 64) {
            resident[0][dev] = sms * (p2 > 0 ? p2 : 1);
            resident[1][dev] = sms * (p3 > 0 ? p3 : 1);
        }
    });
    int dev = 0;
    cudaGetDevice(&dev);
    const int r = (dev >= 0 && dev < 64) ? resident[a.dim == 3][dev] : 0;
    if (r > 0) grid = std::min(grid, r);
    count_launch(1);
    if (a.dim == 2) knn_warp_kernel<2><<<grid, KW_WARPS * 32, 0, st>>>(A);
    else knn_warp_kernel<3><<<grid, KW_WARPS * 32, 0, st>>>(A);
}

}  // namespace zd
