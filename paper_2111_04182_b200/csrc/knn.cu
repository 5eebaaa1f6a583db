// knn.cu — K6 exact k-NN over the zd-tree.
//
// All-points ("leaf-based"): for every live point q, in sorted
// (Morton) order so that neighbouring threads walk neighbouring subtrees:
//   scan q's leaf, then Alg. 3 searchUp: while C has a parent and the
//   k-ball may leave C, run Alg. 2 searchDown on C's sibling, C = parent.
// External queries ("bit-based"): locate the leaf by the query's Morton bits
// from the root, then the same searchUp; nothing is excluded.
//
// Exact rules:
//  * k-best set sorted by (d2, id) in registers (reading 14); a candidate enters iff
//    (d2, id) < the current k-th (reading 11: insert the candidate, not p).
//  * prune a subtree iff boxd2(q, box) > d2 of the k-th (strict; reading 8) — the
//    set starts filled with (INT64_MAX, -1) so "|N| < k" needs no extra test.
//  * stop ascending at C iff q is inside C's tight box and (m+1)^2 > k-th d2,
//    m = min over axes of min(q - lo, hi - q) (reading 9): every point outside
//    subtree(C) lies outside C's Morton cell, which contains the box.
//  * self excluded by id (reading 13); nearer child first by box distance, tie -> left
//    (reading 10; performance only — the answer is unique).
#include <climits>

#include "common.cuh"
#include "internal.h"

namespace zd {

namespace {

template <int K>
struct KBest {
    int64_t d[K];
    int32_t i[K];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int s = 0; s < K; ++s) { d[s] = INT64_MAX; i[s] = -1; }
    }
    __device__ __forceinline__ int64_t worst() const { return d[K - 1]; }
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
    int dx = q.c[0] - r.x, dy = q.c[1] - r.y;
    int64_t s = (int64_t)dx * dx + (int64_t)dy * dy;
    if (DIM == 3) {
        int dz = q.c[2] - r.z;
        s += (int64_t)dz * dz;
    }
    return s;
}

template <int DIM>
__device__ __forceinline__ int64_t boxd2(const Query<DIM>& q, const int32_t* b) {
    int64_t s = 0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        int t = max(b[a] - q.c[a], 0) + max(q.c[a] - b[DIM + a], 0);
        s += (int64_t)t * t;
    }
    return s;
}

// stop test of Alg. 3 (reading 9); false when q is outside the box (external queries)
template <int DIM>
__device__ __forceinline__ bool stop_at(const Query<DIM>& q, const int32_t* b, int64_t worst) {
    int m = INT_MAX;
#pragma unroll
    for (int a = 0; a < DIM; ++a) m = min(m, min(q.c[a] - b[a], b[DIM + a] - q.c[a]));
    if (m < 0) return false;
    const int64_t mm = (int64_t)m + 1;
    return mm * mm > worst;
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

struct Tree {
    const int4* recs;
    const int32_t* leaf_start;
    const int32_t* leaf_parent;
    const void* nodes;
};

template <int DIM, int K>
__device__ __forceinline__ void scan_leaf(const Tree& T, int32_t l, const Query<DIM>& q, KBest<K>& best) {
    const int32_t s = __ldg(T.leaf_start + l), e = __ldg(T.leaf_start + l + 1);
    for (int32_t j = s; j < e; ++j) {
        const int4 r = __ldg(T.recs + j);
        if (r.w == q.id) continue;
        const int64_t d = dist2<DIM>(q, r);
        if (best.accepts(d, r.w)) best.insert(d, r.w);
    }
}

// Alg. 2 searchDown on subtree `sub` whose box is sbox (explicit stack of far children)
template <int DIM, int K>
__device__ __forceinline__ void search_down(const Tree& T, int32_t sub, const int32_t* sbox, const Query<DIM>& q,
                                            KBest<K>& best) {
    if (boxd2<DIM>(q, sbox) > best.worst()) return;
    const Node<DIM>* nodes = static_cast<const Node<DIM>*>(T.nodes);
    int32_t stk_ref[kMaxDepth];
    int64_t stk_d[kMaxDepth];
    int sp = 0;
    int32_t cur = sub;
    while (true) {
        if (is_leaf_ref(cur)) {
            scan_leaf<DIM, K>(T, ~cur, q, best);
        } else {
            const Node<DIM> nd = load_node<DIM>(nodes + cur);
            const int64_t dl = boxd2<DIM>(q, nd.lbox), dr = boxd2<DIM>(q, nd.rbox);
            const bool lfirst = dl <= dr;
            const int64_t dn = lfirst ? dl : dr, df = lfirst ? dr : dl;
            const int64_t w = best.worst();
            if (dn <= w) {
                if (df <= w) {
                    stk_ref[sp] = lfirst ? nd.right : nd.left;
                    stk_d[sp] = df;
                    ++sp;
                }
                cur = lfirst ? nd.left : nd.right;
                continue;
            }
        }
        bool more = false;
        while (sp > 0) {
            --sp;
            if (stk_d[sp] <= best.worst()) { cur = stk_ref[sp]; more = true; break; }
        }
        if (!more) break;
    }
}

// Alg. 3 searchUp from leaf l
template <int DIM, int K>
__device__ __forceinline__ void search_up(const Tree& T, int32_t l, const Query<DIM>& q, KBest<K>& best) {
    const Node<DIM>* nodes = static_cast<const Node<DIM>*>(T.nodes);
    scan_leaf<DIM, K>(T, l, q, best);
    int32_t C = ~l;
    int32_t P = __ldg(T.leaf_parent + l);
    while (P >= 0) {
        const Node<DIM> nd = load_node<DIM>(nodes + P);
        const bool isl = nd.left == C;
        int32_t cb[2 * DIM], sb[2 * DIM];
#pragma unroll
        for (int a = 0; a < 2 * DIM; ++a) {
            cb[a] = isl ? nd.lbox[a] : nd.rbox[a];
            sb[a] = isl ? nd.rbox[a] : nd.lbox[a];
        }
        if (stop_at<DIM>(q, cb, best.worst())) break;
        search_down<DIM, K>(T, isl ? nd.right : nd.left, sb, q, best);
        C = P;
        P = nd.parent;
    }
}

template <int K>
__device__ __forceinline__ void write_row(const KBest<K>& best, int k, int64_t row, int32_t* out_idx, int64_t* out_d2) {
    int32_t* oi = out_idx + row * k;
    int64_t* od = out_d2 + row * k;
#pragma unroll
    for (int s = 0; s < K; ++s) {
        if (s < k) { oi[s] = best.i[s]; od[s] = best.d[s]; }
    }
}

template <int DIM, int K>
__global__ void __launch_bounds__(128) knn_all_kernel(Tree T, const int32_t* __restrict__ pt_leaf, int32_t n, int k,
                                                      const int32_t* __restrict__ row_of_id, int32_t* __restrict__ out_idx,
                                                      int64_t* __restrict__ out_d2) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 r = __ldg(T.recs + i);
    Query<DIM> q;
    q.c[0] = r.x; q.c[1] = r.y; q.c[2] = r.z; q.id = r.w;
    KBest<K> best;
    best.init();
    search_up<DIM, K>(T, __ldg(pt_leaf + i), q, best);
    const int64_t row = row_of_id ? __ldg(row_of_id + r.w) : r.w;
    write_row<K>(best, k, row, out_idx, out_d2);
}

template <int DIM, int K>
__global__ void __launch_bounds__(128) knn_ext_kernel(Tree T, const int32_t* __restrict__ meta,
                                                      const int32_t* __restrict__ queries, int32_t m, int k,
                                                      int32_t* __restrict__ out_idx, int64_t* __restrict__ out_d2) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    Query<DIM> q;
    q.c[2] = 0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) q.c[a] = __ldg(queries + (int64_t)i * DIM + a);
    q.id = -1;
    // bit-based leaf location: follow the query key's bit at each split
    const uint64_t key = morton<DIM>(q.c[0], q.c[1], q.c[2]);
    const Node<DIM>* nodes = static_cast<const Node<DIM>*>(T.nodes);
    int32_t cur = __ldg(meta + 1);
    while (cur >= 0) {
        const int4 tail = __ldg(reinterpret_cast<const int4*>(nodes + cur) + (sizeof(Node<DIM>) / 16 - 1));
        cur = ((key >> tail.w) & 1u) ? tail.y : tail.x;   // (left, right, parent, split)
    }
    KBest<K> best;
    best.init();
    search_up<DIM, K>(T, ~cur, q, best);
    write_row<K>(best, k, i, out_idx, out_d2);
}

template <int DIM, int K>
void launch_all(const KnnArgs& a, cudaStream_t st) {
    Tree T{a.recs, a.leaf_start, a.leaf_parent, a.nodes};
    const int grid = (int)((a.n + 127) / 128);
    if (grid > 0) count_launch(1);
    if (grid > 0)
        knn_all_kernel<DIM, K><<<grid, 128, 0, st>>>(T, a.pt_leaf, (int32_t)a.n, a.k, a.row_of_id, a.out_idx, a.out_d2);
}

template <int DIM, int K>
void launch_ext(const KnnArgs& a, const int32_t* queries, int64_t m, cudaStream_t st) {
    Tree T{a.recs, a.leaf_start, a.leaf_parent, a.nodes};
    const int grid = (int)((m + 127) / 128);
    if (grid > 0) count_launch(1);
    if (grid > 0) knn_ext_kernel<DIM, K><<<grid, 128, 0, st>>>(T, a.d_meta, queries, (int32_t)m, a.k, a.out_idx, a.out_d2);
}

#define ZD_K_CASES(X) X(1) X(4) X(8) X(10) X(16) X(32)

template <int DIM>
void all_dim(const KnnArgs& a, cudaStream_t st) {
#define X(KK) if (a.k <= KK) { launch_all<DIM, KK>(a, st); return; }
    ZD_K_CASES(X)
#undef X
}

template <int DIM>
void ext_dim(const KnnArgs& a, const int32_t* queries, int64_t m, cudaStream_t st) {
#define X(KK) if (a.k <= KK) { launch_ext<DIM, KK>(a, queries, m, st); return; }
    ZD_K_CASES(X)
#undef X
}

}  // namespace

int knn_kmax() { return 32; }

void knn_all(const KnnArgs& a, cudaStream_t st) {
    if (a.dim == 2) all_dim<2>(a, st); else all_dim<3>(a, st);
}

void knn_queries(const KnnArgs& a, const int32_t* queries, int64_t m, int* d_invalid, cudaStream_t st) {
    (void)d_invalid;
    if (a.dim == 2) ext_dim<2>(a, queries, m, st); else ext_dim<3>(a, queries, m, st);
}

}  // namespace zd
