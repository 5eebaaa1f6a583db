// api.cu — the C ABI of include/zd.h: handle, device memory, stream, orchestration.
//
// Host side only launches kernels (sort.cu, tree.cu, knn.cu, update.cu); every step
// of the hot path runs on the GPU.  Memory comes from a private stream-ordered pool per
// device (cudaMallocFromPoolAsync) with the release threshold raised, so repeated
// builds and updates reuse memory without device-wide synchronisation; zd_trim()
// returns the cached memory.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <mutex>
#include <vector>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "../../include/zd.h"
#include "internal.h"

using namespace zd;

namespace zd {
static std::atomic<int64_t> g_launches{0};
void count_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

static PerDeviceOnce g_pool_once;
static cudaMemPool_t g_pools[64] = {};

static cudaMemPool_t device_pool() {
    g_pool_once.run([](int dev) {
        if (const char* e = std::getenv("ZD_POOL"); e && !std::strcmp(e, "default")) {   // testing
            cudaMemPool_t dp = nullptr;
            if (cudaDeviceGetDefaultMemPool(&dp, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(dp, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            return;
        }
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            g_pools[dev & 63] = pool;
        } else {
            cudaGetLastError();   // fall back to the default pool
        }
    });
    int dev = 0;
    cudaGetDevice(&dev);
    return g_pools[dev & 63];
}

cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t st) {
    cudaMemPool_t pool = device_pool();
    return pool ? cudaMallocFromPoolAsync(p, bytes, pool, st) : cudaMallocAsync(p, bytes, st);
}
}  // namespace zd

namespace {

thread_local std::string g_err;
thread_local int g_err_code = 0;

int fail(int code, const std::string& msg) {
    g_err = msg;
    g_err_code = code;
    return code;
}

void clear_err() {
    g_err.clear();
    g_err_code = 0;
}

// NVTX range over a C-ABI call or one of its phases (SURVEY §5 tracing): free when no
// profiler is attached (NVTX3 is header-only; nsys / ncu --nvtx pick the ranges up).
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

// Runs a cleanup at scope exit (scratch of an update that returns early on an error).
template <class F>
struct ScopeExit {
    F f;
    ~ScopeExit() { f(); }
};
template <class F>
ScopeExit<F> at_exit(F f) { return ScopeExit<F>{f}; }

int cuda_fail(cudaError_t e, const char* where) {
    cudaGetLastError();   // clear sticky-free errors
    const int code = (e == cudaErrorMemoryAllocation) ? ZD_ENOMEM : ZD_ECUDA;
    return fail(code, std::string(where) + ": " + cudaGetErrorString(e));
}

#define ZD_CUDA(call)                                              \
    do {                                                           \
        cudaError_t e_ = (call);                                   \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);        \
    } while (0)

#define ZD_CHECK_LAUNCH(where)                                     \
    do {                                                           \
        cudaError_t e_ = cudaGetLastError();                       \
        if (e_ != cudaSuccess) return cuda_fail(e_, where);        \
    } while (0)

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <class T>
cudaError_t dalloc(T** p, size_t count, cudaStream_t st) {
    *p = nullptr;
    if (count == 0) count = 1;
    return pool_alloc((void**)p, count * sizeof(T), st);
}

template <class T>
void dfree(T*& p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
}

// Process-wide pinned host arena of small per-handle mailboxes (one cudaMallocHost
// for the process instead of one per handle).
struct PinnedSlots {
    static constexpr int kSlots = 4096, kWords = 8;
    std::mutex mu;
    int32_t* base = nullptr;
    std::vector<int> free_list;
    int32_t* get() {
        std::lock_guard<std::mutex> g(mu);
        if (!base) {
            if (cudaMallocHost((void**)&base, sizeof(int32_t) * kSlots * kWords) != cudaSuccess) {
                cudaGetLastError();
                base = nullptr;
                return nullptr;
            }
            for (int i = kSlots - 1; i >= 0; --i) free_list.push_back(i);
        }
        if (free_list.empty()) return nullptr;
        int s = free_list.back();
        free_list.pop_back();
        return base + (size_t)s * kWords;
    }
    bool put(int32_t* p) {
        std::lock_guard<std::mutex> g(mu);
        if (!base || p < base || p >= base + (size_t)kSlots * kWords) return false;
        free_list.push_back((int)((p - base) / kWords));
        return true;
    }
};
PinnedSlots& pinned() {
    static PinnedSlots* p = new PinnedSlots();   // never destroyed (process lifetime)
    return *p;
}

enum Phase { PH_SORT = 0, PH_TOPO = 1, PH_BBOX = 2, PH_MERGE = 3, PH_KNN = 4, PH_VALID = 5, NPH = 6 };

}  // namespace

struct zd_tree {
    int dim = 3, leaf_max = 16;
    cudaStream_t st = nullptr;
    int64_t n = 0, n_next = 0, cap = 0, id_cap = 0;
    int64_t ncap = 0;   // internal-node capacity of the node-indexed tree buffers
    int64_t fast_inserts = 0;   // inserts applied by the NEXT-2 fast path (introspection/tests)
    int64_t fast_deletes = 0;   // deletes applied by the NEXT-2 fast path
    int64_t trunc_fallbacks = 0;   // builds whose truncated sort had to be redone with all passes
    bool shift_set = false;
    int32_t shift[3] = {0, 0, 0};   // random shift, applied before encoding
    // sorted live points
    uint64_t* keys = nullptr;
    int4* recs = nullptr;
    uint64_t* keys2 = nullptr;
    int4* recs2 = nullptr;
    TreeBufs tb{};
    // id bookkeeping
    uint32_t* alive = nullptr;     // [id_cap/32] bitset
    int32_t* row_of_id = nullptr;  // [id_cap]
    int32_t* live_ids = nullptr;   // [cap]
    uint32_t* rank_cnt = nullptr;  // [rank_blocks(id_cap)+1]
    bool rows_identity = true, rows_dirty = false;
    // small scratch
    int32_t* d_small = nullptr;    // [0..3] meta copy area, [4] invalid flag, [6..7] u64 count
    int32_t* h_small = nullptr;    // pinned mirror
    // timing
    bool timing = false;
    cudaEvent_t ev[8] = {};
    float ms[NPH] = {};
    bool host_meta_valid = false;
    int64_t n_leaves = 1, n_internal = 0;
    int32_t root = ~0;
    std::mutex mu;   // guards ms[PH_KNN] written by concurrent zd_knn calls
    // set while an update mutates the handle; left set if the update fails half-way
    // (e.g. ENOMEM in the topology rebuild), after which every call refuses the handle
    bool poisoned = false;
};

namespace {

int* d_invalid(zd_tree* h) { return h->d_small + 4; }

// NULL or poisoned handles are refused (ZD_EINVAL / ZD_ECUDA).
int check_handle(const zd_tree* h) {
    if (!h) return fail(ZD_EINVAL, "NULL handle");
    if (h->poisoned) return fail(ZD_ECUDA, "handle unusable: an earlier update failed half-way (free it)");
    return ZD_OK;
}
unsigned long long* d_count(zd_tree* h) { return reinterpret_cast<unsigned long long*>(h->d_small + 6); }

void free_tree_bufs(zd_tree* h) {
    TreeBufs& t = h->tb;
    dfree(t.pt_leaf, h->st); dfree(t.leaf_start, h->st); dfree(t.leaf_parent, h->st);
    dfree(t.split_bit, h->st); dfree(t.visit, h->st); dfree(t.range, h->st); dfree(t.pos_range, h->st);
    dfree(t.flags, h->st); dfree(t.block_cnt, h->st);
    if (t.nodes) { cudaFreeAsync(t.nodes, h->st); t.nodes = nullptr; }
    h->ncap = 0;
}

// Node-indexed buffers (internal nodes <= ncap, leaves <= ncap + 1).
void free_node_bufs(zd_tree* h) {
    TreeBufs& t = h->tb;
    dfree(t.leaf_start, h->st); dfree(t.leaf_parent, h->st); dfree(t.split_bit, h->st);
    dfree(t.visit, h->st); dfree(t.range, h->st); dfree(t.pos_range, h->st);
    if (t.nodes) { cudaFreeAsync(t.nodes, h->st); t.nodes = nullptr; }
    h->ncap = 0;
}
int alloc_node_bufs(zd_tree* h, int64_t ncap) {
    free_node_bufs(h);
    TreeBufs& t = h->tb;
    ncap = std::max<int64_t>(ncap, 1);
    const size_t node_bytes = h->dim == 2 ? 48 : 64;
    ZD_CUDA(dalloc(&t.leaf_start, ncap + 2, h->st));
    ZD_CUDA(dalloc(&t.leaf_parent, ncap + 1, h->st));
    ZD_CUDA(dalloc(&t.split_bit, ncap, h->st));
    ZD_CUDA(dalloc(&t.visit, ncap, h->st));
    ZD_CUDA(dalloc(&t.range, 2 * ncap, h->st));
    ZD_CUDA(dalloc(&t.pos_range, ncap, h->st));
    ZD_CUDA(pool_alloc(&t.nodes, ncap * node_bytes, h->st));
    h->ncap = ncap;
    return ZD_OK;
}

// Below this many points the node buffers are sized for the worst case (n - 1
// internal nodes) and the topology needs no host round trip; above it they are sized
// from the node count of each build (one sync after the flag scan), so the tree takes
// ~14 B/pt instead of ~100 (3D, leaf size 16) and 10^9 points fit in 180 GB.
// ZD_EXACT_NODES_MIN (testing) overrides the threshold.
int64_t exact_nodes_min() {
    if (const char* e = std::getenv("ZD_EXACT_NODES_MIN")) return std::atoll(e);
    return (int64_t)1 << 25;
}

int alloc_tree_bufs(zd_tree* h, int64_t cap) {
    free_tree_bufs(h);
    TreeBufs& t = h->tb;
    t.d_meta = h->d_small;
    ZD_CUDA(dalloc(&t.pt_leaf, cap, h->st));
    ZD_CUDA(dalloc(&t.flags, cap, h->st));
    ZD_CUDA(dalloc(&t.block_cnt, std::max(tree_blocks(cap), compact_blocks(cap)) + 2, h->st));
    return alloc_node_bufs(h, cap <= exact_nodes_min() ? cap : cap / 8);
}

// Point capacity for keys/recs (and their alternates) + tree buffers.  With
// old_keys/old_recs the current primary arrays are handed back to the caller (still
// allocated; it reads them once, e.g. as the merge source, then frees them) instead
// of being copied into the new ones.
int ensure_point_cap(zd_tree* h, int64_t need, uint64_t** old_keys = nullptr, int4** old_recs = nullptr,
                     bool keep_nodes = false) {
    if (need <= h->cap && h->keys) return ZD_OK;
    const int64_t cap = std::max<int64_t>(need, h->cap + h->cap / 4);
    uint64_t* nk = nullptr;
    int4* nr = nullptr;
    ZD_CUDA(dalloc(&nk, cap, h->st));
    ZD_CUDA(dalloc(&nr, cap, h->st));
    if (old_keys) {
        *old_keys = h->keys;
        *old_recs = h->recs;
        h->keys = nullptr;
        h->recs = nullptr;
    }
    dfree(h->keys, h->st); dfree(h->recs, h->st); dfree(h->keys2, h->st); dfree(h->recs2, h->st);
    dfree(h->live_ids, h->st);
    h->keys = nk;
    h->recs = nr;
    ZD_CUDA(dalloc(&h->keys2, cap, h->st));
    ZD_CUDA(dalloc(&h->recs2, cap, h->st));
    ZD_CUDA(dalloc(&h->live_ids, cap, h->st));
    h->cap = cap;
    h->rows_dirty = true;   // live_ids was reallocated
    if (keep_nodes && h->tb.nodes) {
        // the insert fast path keeps the node-indexed buffers: only the point-indexed
        // ones grow (their contents are rewritten by the fast path)
        TreeBufs& t = h->tb;
        dfree(t.pt_leaf, h->st); dfree(t.flags, h->st); dfree(t.block_cnt, h->st);
        ZD_CUDA(dalloc(&t.pt_leaf, cap, h->st));
        ZD_CUDA(dalloc(&t.flags, cap, h->st));
        ZD_CUDA(dalloc(&t.block_cnt, std::max(tree_blocks(cap), compact_blocks(cap)) + 2, h->st));
        return ZD_OK;
    }
    return alloc_tree_bufs(h, cap);
}

int ensure_id_cap(zd_tree* h, int64_t need) {
    if (need <= h->id_cap && h->alive) return ZD_OK;
    const int64_t cap = std::max<int64_t>(need, h->id_cap + h->id_cap / 4);
    const int64_t words = (cap + 31) / 32, old_words = (h->id_cap + 31) / 32;
    uint32_t* na = nullptr;
    ZD_CUDA(dalloc(&na, words, h->st));
    ZD_CUDA(cudaMemsetAsync(na, 0, words * sizeof(uint32_t), h->st));
    if (h->alive && old_words > 0)
        ZD_CUDA(cudaMemcpyAsync(na, h->alive, old_words * sizeof(uint32_t), cudaMemcpyDeviceToDevice, h->st));
    dfree(h->alive, h->st);
    dfree(h->row_of_id, h->st);
    dfree(h->rank_cnt, h->st);
    h->alive = na;
    ZD_CUDA(dalloc(&h->row_of_id, cap, h->st));
    ZD_CUDA(dalloc(&h->rank_cnt, rank_blocks(cap) + 2, h->st));
    h->id_cap = cap;
    h->rows_dirty = true;
    return ZD_OK;
}

// Sorted (keys, recs) of n points with ids id_base.. into the given outputs.
// use_alt: the ping-pong buffers live in the idle update alternates keys2/recs2
// (8 + 16 bytes per point = 2 x (u64 key + u32 id)); else they are allocated.
int sort_into(zd_tree* h, const int32_t* dpts, int64_t n, uint32_t id_base, uint64_t* keys_out, int4* recs_out,
              bool use_alt = false, int* d_trunc_fail = nullptr, bool approx = false) {
    if (n <= 0) return ZD_OK;
    Nvtx range("encode+radix sort");
    if (n <= kSmallSort) {   // small batches: one rank-by-counting launch (sort.cu)
        sort_points_small(h->dim, dpts, n, id_base, keys_out, recs_out, d_invalid(h), h->st,
                          h->shift_set ? h->shift : nullptr);
        ZD_CHECK_LAUNCH("sort_points_small");
        return ZD_OK;
    }
    SortScratch s{};
    const bool alt = use_alt && h->keys2 && h->recs2 && n <= h->cap;
    if (alt) {
        s.k[0] = h->keys2;
        s.k[1] = reinterpret_cast<uint64_t*>(h->recs2);
        s.v[0] = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(h->recs2) + (size_t)n * sizeof(uint64_t));
        s.v[1] = s.v[0] + n;
    } else {
        ZD_CUDA(dalloc(&s.k[0], n, h->st));
        ZD_CUDA(dalloc(&s.k[1], n, h->st));
        ZD_CUDA(dalloc(&s.v[0], n, h->st));
        ZD_CUDA(dalloc(&s.v[1], n, h->st));
    }
    s.zero_words = sort_zero_words(n);
    ZD_CUDA(dalloc(&s.zero_block, s.zero_words, h->st));
    ZD_CUDA(dalloc(&s.offs, 8 * 256, h->st));
    sort_points(h->dim, dpts, n, id_base, keys_out, recs_out, s, d_invalid(h), h->st, h->shift_set ? h->shift : nullptr,
                d_trunc_fail, approx);
    ZD_CHECK_LAUNCH("sort_points");
    if (!alt) { dfree(s.k[0], h->st); dfree(s.k[1], h->st); dfree(s.v[0], h->st); dfree(s.v[1], h->st); }
    dfree(s.zero_block, h->st); dfree(s.offs, h->st);
    return ZD_OK;
}

void rec(zd_tree* h, int i) {
    if (h->timing) cudaEventRecord(h->ev[i], h->st);
}

void elapsed(zd_tree* h, int phase, int a, int b) {
    float t = 0.f;
    if (h->timing && cudaEventElapsedTime(&t, h->ev[a], h->ev[b]) == cudaSuccess) h->ms[phase] = t;
}

// Builds of at least this many points use the truncated sort (sort.cu); ZD_SORT_TRUNC=0
// disables it (testing).
constexpr int64_t kTruncSortMin = (int64_t)1 << 20;
bool trunc_enabled() {
    const char* e = std::getenv("ZD_SORT_TRUNC");
    return !(e && e[0] == '0');
}

// Largest key count of one radix sort (sort.cu: 30-bit digit counts in the look-back
// status words).  Builds, insert batches and external query sets stay below it.
constexpr int64_t kMaxSortKeys = (int64_t)1 << 30;

// NEXT-2 insert fast path: batches up to this size are checked; ZD_INCR=0 disables it.
constexpr int64_t kIncrMaxBatch = (int64_t)1 << 16;
bool incr_enabled() {
    const char* e = std::getenv("ZD_INCR");
    return !(e && e[0] == '0');
}

int topology(zd_tree* h) {
    Nvtx range("topology+boxes");
    if (h->ncap < h->n - 1) {
        // node buffers sized by count: flag + scan, read the internal-node count, grow
        topology_flags(h->keys, h->n, h->leaf_max, h->tb, h->st);
        ZD_CHECK_LAUNCH("topology_flags");
        ZD_CUDA(cudaMemcpyAsync(h->h_small + 2, h->tb.block_cnt + tree_blocks(h->n), sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, h->st));
        ZD_CUDA(cudaStreamSynchronize(h->st));
        const int64_t nb = (int64_t)(uint32_t)h->h_small[2];
        if (nb > h->ncap) {
            int rc = alloc_node_bufs(h, std::min<int64_t>(h->n - 1, nb + nb / 8));
            if (rc) return rc;
        }
        topology_finish(h->dim, h->keys, h->recs, h->n, h->tb, h->st, h->timing ? h->ev[6] : nullptr);
    } else {
        build_topology(h->dim, h->keys, h->recs, h->n, h->leaf_max, h->tb, h->st, h->timing ? h->ev[6] : nullptr);
    }
    ZD_CHECK_LAUNCH("build_topology");
    h->host_meta_valid = false;
    return ZD_OK;
}

int sync_meta(zd_tree* h) {
    ZD_CUDA(cudaMemcpyAsync(h->h_small, h->d_small, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, h->st));
    ZD_CUDA(cudaStreamSynchronize(h->st));
    return ZD_OK;
}

int refresh_host_meta(zd_tree* h) {
    if (h->host_meta_valid) return ZD_OK;
    int rc = sync_meta(h);
    if (rc) return rc;
    h->n_internal = h->h_small[0];
    h->n_leaves = h->n_internal + 1;
    h->root = h->h_small[1];
    h->host_meta_valid = true;
    return ZD_OK;
}

int ensure_rows(zd_tree* h) {
    if (h->rows_identity || !h->rows_dirty) return ZD_OK;
    rank_alive(h->alive, h->n_next, h->row_of_id, h->live_ids, h->rank_cnt, h->st);
    ZD_CHECK_LAUNCH("rank_alive");
    h->rows_dirty = false;
    return ZD_OK;
}

// Device copy of a caller array (host or device).  *owned is set when staged.
int stage_in(zd_tree* h, const void* src, size_t bytes, const void** dev, void** owned) {
    *owned = nullptr;
    if (bytes == 0 || is_device_ptr(src)) { *dev = src; return ZD_OK; }
    void* d = nullptr;
    ZD_CUDA(pool_alloc(&d, bytes, h->st));
    ZD_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, h->st));
    *owned = d;
    *dev = d;
    return ZD_OK;
}

void destroy(zd_tree* h) {
    if (!h) return;
    dfree(h->keys, h->st); dfree(h->recs, h->st); dfree(h->keys2, h->st); dfree(h->recs2, h->st);
    free_tree_bufs(h);
    dfree(h->alive, h->st); dfree(h->row_of_id, h->st); dfree(h->live_ids, h->st); dfree(h->rank_cnt, h->st);
    dfree(h->d_small, h->st);
    cudaStreamSynchronize(h->st);
    if (h->h_small && !pinned().put(h->h_small)) delete[] h->h_small;
    for (auto& e : h->ev) if (e) cudaEventDestroy(e);
    delete h;
}

int do_build(zd_tree* h, const int32_t* points, int64_t n) {
    ZD_CUDA(dalloc(&h->d_small, 8, h->st));
    h->h_small = pinned().get();
    if (!h->h_small) h->h_small = new int32_t[8];
    if (h->timing) for (auto& e : h->ev) ZD_CUDA(cudaEventCreate(&e));
    ZD_CUDA(cudaMemsetAsync(h->d_small, 0, 8 * sizeof(int32_t), h->st));
    const void* dpts = nullptr;
    void* owned = nullptr;
    int rc = stage_in(h, points, (size_t)n * h->dim * sizeof(int32_t), &dpts, &owned);
    if (rc) return rc;
    if ((rc = ensure_point_cap(h, std::max<int64_t>(n, 1)))) return rc;
    if ((rc = ensure_id_cap(h, std::max<int64_t>(n, 1)))) return rc;
    h->n = n;
    h->n_next = n;
    // large builds sort with 5 passes + a run fixup; its verdict is read at the one sync
    // (d_small[3]) and a failed fixup (runs of > 64 equal 40-bit prefixes: degenerate
    // inputs) redoes the sort and topology with all 8 passes
    const bool trunc = n >= kTruncSortMin && trunc_enabled();
    rec(h, 0);
    if ((rc = sort_into(h, (const int32_t*)dpts, n, 0, h->keys, h->recs, true, trunc ? h->d_small + 3 : nullptr)))
        return rc;
    rec(h, 1);
    if ((rc = topology(h))) return rc;
    rec(h, 2);
    set_alive_range(h->alive, 0, n, h->st);
    h->rows_identity = true;
    if ((rc = refresh_host_meta(h))) return rc;   // the one sync: validation flag + node count
    if (trunc && h->h_small[3] && !h->h_small[4]) {
        h->trunc_fallbacks += 1;
        rec(h, 0);
        if ((rc = sort_into(h, (const int32_t*)dpts, n, 0, h->keys, h->recs, true))) return rc;
        rec(h, 1);
        if ((rc = topology(h))) return rc;
        rec(h, 2);
        if ((rc = refresh_host_meta(h))) return rc;
    }
    if (owned) cudaFreeAsync(owned, h->st);
    elapsed(h, PH_SORT, 0, 1);
    elapsed(h, PH_TOPO, 1, 6);
    elapsed(h, PH_BBOX, 6, 2);
    if (h->h_small[4]) return fail(ZD_ERANGE, "zd_build: coordinate outside the universe box [0, 2^B)");
    return ZD_OK;
}

int knn_impl(zd_tree* h, const int32_t* queries, int64_t m, int k, int32_t* out_idx, int64_t* out_dist2, int flags,
             int64_t q_lo, int64_t q_hi);

}  // namespace

extern "C" {

const char* zd_last_error(void) { return g_err.c_str(); }
int zd_last_error_code(void) { return g_err_code; }

zd_tree* zd_build_ex(const int32_t* points, int64_t n, int dim, const zd_opts* opts) {
    Nvtx range("zd_build");
    clear_err();
    if (dim != 2 && dim != 3) { fail(ZD_EINVAL, "zd_build: dim must be 2 or 3"); return nullptr; }
    // the radix sort's look-back words carry 30-bit digit counts: one sort holds < 2^30 keys
    if (n < 0 || n >= kMaxSortKeys) { fail(ZD_EINVAL, "zd_build: need 0 <= n < 2^30"); return nullptr; }
    if (n > 0 && !points) { fail(ZD_EINVAL, "zd_build: points is NULL"); return nullptr; }
    int leaf_max = 16;
    cudaStream_t st = nullptr;
    if (opts) {
        if (opts->leaf_max) leaf_max = opts->leaf_max;
        st = (cudaStream_t)opts->stream;
    }
    const bool timing = opts && opts->timing;
    if (leaf_max < 1 || leaf_max > ZD_LEAF_MAX_MAX) { fail(ZD_EINVAL, "zd_build: leaf_max out of range"); return nullptr; }
    const bool shift_set = opts && opts->shift_set;
    if (shift_set) {
        const int lim = dim == 2 ? (1 << 30) : (1 << 21);   // shifted axes: 31 / 22 bits
        for (int a = 0; a < dim; ++a)
            if (opts->shift[a] < 0 || opts->shift[a] >= lim) {
                fail(ZD_EINVAL, dim == 2 ? "zd_build: shift outside [0, 2^30)" : "zd_build: shift outside [0, 2^21)");
                return nullptr;
            }
    }
    zd_tree* h = new zd_tree();
    h->dim = dim;
    h->leaf_max = leaf_max;
    h->st = st;
    h->timing = timing;
    if (shift_set) {
        h->shift_set = true;
        for (int a = 0; a < dim; ++a) h->shift[a] = opts->shift[a];
    }
    if (do_build(h, points, n) != ZD_OK) {
        std::string e = g_err;
        int c = g_err_code;
        destroy(h);
        fail(c, e);
        return nullptr;
    }
    return h;
}

zd_tree* zd_build(const int32_t* points, int64_t n, int dim) { return zd_build_ex(points, n, dim, nullptr); }

void zd_free(zd_tree* h) { destroy(h); }

int64_t zd_size(const zd_tree* h) { return h ? h->n : fail(ZD_EINVAL, "NULL handle"); }

int zd_set_stream(zd_tree* h, void* stream) {
    if (!h) return fail(ZD_EINVAL, "NULL handle");
    ZD_CUDA(cudaStreamSynchronize(h->st));
    h->st = (cudaStream_t)stream;
    return ZD_OK;
}

int zd_set_timing(zd_tree* h, int enable) {
    if (!h) return fail(ZD_EINVAL, "NULL handle");
    if (enable && !h->ev[0])
        for (auto& e : h->ev) ZD_CUDA(cudaEventCreate(&e));
    h->timing = enable != 0;
    return ZD_OK;
}

int64_t zd_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int zd_trim(void) {
    clear_err();
    cudaMemPool_t pool = device_pool();
    if (!pool) return ZD_OK;
    ZD_CUDA(cudaDeviceSynchronize());   // frees still pending on streams complete first
    ZD_CUDA(cudaMemPoolTrimTo(pool, 0));
    return ZD_OK;
}

int zd_knn_stats(int64_t* out, int n, int reset) {
    clear_err();
    if (!out || n < 0) return fail(ZD_EINVAL, "zd_knn_stats: bad arguments");
    const int r = knn_stats(reinterpret_cast<unsigned long long*>(out), n, reset);
    if (r < 0) return fail(ZD_EINVAL, "zd_knn_stats: not a -DZD_KNN_STATS build");
    return r;
}

int zd_get_timing(const zd_tree* h, float* ms, int nphase) {
    if (!h || !ms) return fail(ZD_EINVAL, "NULL argument");
    int c = std::min(nphase, (int)NPH);
    for (int i = 0; i < c; ++i) ms[i] = h->ms[i];
    return c;
}

int zd_knn(zd_tree* h, const int32_t* queries, int64_t m, int k, int32_t* out_idx, int64_t* out_dist2) {
    return zd_knn_ex(h, queries, m, k, out_idx, out_dist2, 0);
}

int zd_knn_ex(zd_tree* h, const int32_t* queries, int64_t m, int k, int32_t* out_idx, int64_t* out_dist2, int flags) {
    clear_err();
    return knn_impl(h, queries, m, k, out_idx, out_dist2, flags, 0, h ? h->n : 0);
}

int zd_knn_range(zd_tree* h, int64_t pos_lo, int64_t pos_hi, int k, int32_t* out_idx, int64_t* out_dist2, int flags) {
    clear_err();
    if (int e = check_handle(h)) return e;
    if (pos_lo < 0 || pos_hi < pos_lo || pos_hi > h->n) return fail(ZD_EINVAL, "zd_knn_range: need 0 <= pos_lo <= pos_hi <= zd_size(h)");
    if (pos_hi > pos_lo && (!is_device_ptr(out_idx) || !is_device_ptr(out_dist2)))
        return fail(ZD_EINVAL, "zd_knn_range: outputs must be device arrays [zd_size(h)][k]");
    return knn_impl(h, nullptr, h->n, k, out_idx, out_dist2, flags, pos_lo, pos_hi);
}

}  // extern "C"

namespace {

int knn_impl(zd_tree* h, const int32_t* queries, int64_t m, int k, int32_t* out_idx, int64_t* out_dist2, int flags,
             int64_t q_lo, int64_t q_hi) {
    Nvtx range(queries ? "zd_knn(queries)" : "zd_knn(all points)");
    if (flags & ~(ZD_KNN_ROOT_BASED | ZD_KNN_WARP)) return fail(ZD_EINVAL, "zd_knn_ex: unknown flags");
    if (int e = check_handle(h)) return e;
    if (k < 1 || k > ZD_K_MAX) return fail(ZD_EINVAL, "zd_knn: k must be in [1, ZD_K_MAX]");
    if (m < 0 || (queries ? m >= kMaxSortKeys : m >= ((int64_t)1 << 31) - 1))
        return fail(ZD_EINVAL, "zd_knn: bad m (external queries: m < 2^30)");
    if (!queries && m != h->n) return fail(ZD_EINVAL, "zd_knn: all-points query needs m == zd_size(h)");
    if (m > 0 && (!out_idx || !out_dist2)) return fail(ZD_EINVAL, "zd_knn: NULL output");
    if (m == 0 || (!queries && q_hi <= q_lo)) return ZD_OK;   // (an empty shard writes nothing)
    int rc;
    // Outputs: device pointers are written directly; host buffers are staged through
    // device memory and copied back (rows land scattered by id, so writing them over
    // PCIe from the kernel is ~12x slower than one bulk copy, measured).
    int32_t* di = out_idx;
    int64_t* dd = out_dist2;
    const bool host_out = !is_device_ptr(out_idx) || !is_device_ptr(out_dist2);
    if (host_out) {
        ZD_CUDA(dalloc(&di, (size_t)m * k, h->st));
        ZD_CUDA(dalloc(&dd, (size_t)m * k, h->st));
    }
    // scratch for packets deferred to the k-NN second pass (knn.cu): a count + a list
    constexpr int kHardCap = 1 << 15;
    int32_t* hard = nullptr;
    ZD_CUDA(dalloc(&hard, kHardCap + 2, h->st));
    ZD_CUDA(cudaMemsetAsync(hard, 0, 2 * sizeof(int32_t), h->st));   // [0] deferred count, [1] packet counter
    KnnArgs a{};
    a.hard_count = hard;
    a.hard_list = hard + 2;
    a.hard_cap = kHardCap;
    a.root_based = (flags & ZD_KNN_ROOT_BASED) ? 1 : 0;
    a.warp = (flags & ZD_KNN_WARP) ? 1 : 0;
    // ZD_KNN_DEFER (testing): "none" = no second pass, "all" = every packet deferred
    // (up to the list capacity); default: incoherent packets only
    if (const char* dm = std::getenv("ZD_KNN_DEFER")) {
        if (!std::strcmp(dm, "none")) a.hard_list = nullptr;
        else if (!std::strcmp(dm, "all")) a.defer_all = 1;
    }
    a.dim = h->dim; a.k = k; a.n = h->n;
    a.q_lo = q_lo; a.q_hi = q_hi;
    a.recs = h->recs; a.pt_leaf = h->tb.pt_leaf; a.leaf_start = h->tb.leaf_start;
    a.leaf_parent = h->tb.leaf_parent; a.nodes = h->tb.nodes; a.node_range = h->tb.range;
    a.pos_range = h->tb.pos_range;
    a.split_bit = h->tb.split_bit;
    a.d_meta = h->d_small;
    a.out_idx = di; a.out_d2 = dd;
    // zd_knn only reads the handle (concurrent calls are allowed): the row map is
    // refreshed by the mutators, timing uses events of this call
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (h->timing) {
        ZD_CUDA(cudaEventCreate(&ev0));
        ZD_CUDA(cudaEventCreate(&ev1));
    }
    if (!queries) {
        a.row_of_id = h->rows_identity ? nullptr : h->row_of_id;
        if (ev0) cudaEventRecord(ev0, h->st);
        knn_all(a, h->st);
        ZD_CHECK_LAUNCH("knn_all");
        if (ev1) cudaEventRecord(ev1, h->st);
    } else {
        const void* dq = nullptr;
        void* owned = nullptr;
        if ((rc = stage_in(h, queries, (size_t)m * h->dim * sizeof(int32_t), &dq, &owned))) return rc;
        ZD_CUDA(cudaMemsetAsync(d_invalid(h), 0, sizeof(int), h->st));
        validate_points(h->dim, (const int32_t*)dq, m, d_invalid(h), h->st);
        ZD_CUDA(cudaMemcpyAsync(h->h_small + 4, d_invalid(h), sizeof(int), cudaMemcpyDeviceToHost, h->st));
        ZD_CUDA(cudaStreamSynchronize(h->st));
        if (h->h_small[4]) {
            if (owned) cudaFreeAsync(owned, h->st);
            if (host_out) { dfree(di, h->st); dfree(dd, h->st); }
            dfree(hard, h->st);
            return fail(ZD_ERANGE, "zd_knn: query outside the universe box");
        }
        // Morton-sort the queries (K1/K2; ids = query index), locate their leaves by
        // their key bits and run the packet search in Morton order
        uint64_t* qk = nullptr;
        int4* qr = nullptr;
        int32_t* ql = nullptr;
        ZD_CUDA(dalloc(&qk, m, h->st));
        ZD_CUDA(dalloc(&qr, m, h->st));
        ZD_CUDA(dalloc(&ql, m, h->st));
        if (ev0) cudaEventRecord(ev0, h->st);
        // the queries' order only serves locality (the answer does not depend on it):
        // sort them by key bits 24..63 (5 passes)
        if ((rc = sort_into(h, (const int32_t*)dq, m, 0, qk, qr, false, nullptr, true))) return rc;
        knn_queries(a, qk, qr, ql, m, h->st);
        ZD_CHECK_LAUNCH("knn_queries");
        if (ev1) cudaEventRecord(ev1, h->st);
        if (owned) cudaFreeAsync(owned, h->st);
        dfree(qk, h->st);
        dfree(qr, h->st);
        dfree(ql, h->st);
    }
    dfree(hard, h->st);
    if (host_out) {
        ZD_CUDA(cudaMemcpyAsync(out_idx, di, (size_t)m * k * sizeof(int32_t), cudaMemcpyDeviceToHost, h->st));
        ZD_CUDA(cudaMemcpyAsync(out_dist2, dd, (size_t)m * k * sizeof(int64_t), cudaMemcpyDeviceToHost, h->st));
        dfree(di, h->st);
        dfree(dd, h->st);
        ZD_CUDA(cudaStreamSynchronize(h->st));
    }
    if (ev0) {
        float t = 0.f;
        ZD_CUDA(cudaEventSynchronize(ev1));
        if (cudaEventElapsedTime(&t, ev0, ev1) == cudaSuccess) {
            std::lock_guard<std::mutex> g(h->mu);
            h->ms[PH_KNN] = t;
        }
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
    }
    return ZD_OK;
}

}  // namespace

extern "C" {

int64_t zd_insert(zd_tree* h, const int32_t* batch, int64_t m) {
    Nvtx range("zd_insert");
    clear_err();
    if (int e = check_handle(h)) return e;
    if (m < 0 || m >= kMaxSortKeys) return fail(ZD_EINVAL, "zd_insert: need 0 <= m < 2^30");
    if (m == 0) return h->n_next;
    if (!batch) return fail(ZD_EINVAL, "zd_insert: batch is NULL");
    if (h->n_next + m >= ((int64_t)1 << 31) - 1) return fail(ZD_EINVAL, "zd_insert: id space exhausted (2^31)");
    int rc;
    const void* db = nullptr;
    void* owned = nullptr;
    if ((rc = stage_in(h, batch, (size_t)m * h->dim * sizeof(int32_t), &db, &owned))) return rc;
    // validation before any mutation; the batch is sorted into scratch and the
    // fast-path check runs before the one sync, which reads the validation flag, the
    // check's verdict and the node meta together
    rec(h, 0);
    ZD_CUDA(cudaMemsetAsync(d_invalid(h), 0, 2 * sizeof(int), h->st));   // [4] invalid, [5] fast path refused
    validate_points(h->dim, (const int32_t*)db, m, d_invalid(h), h->st);
    rec(h, 1);
    const int64_t first = h->n_next;
    // sorted batch with ids first.. (K7)
    uint64_t* bk = nullptr;
    int4* br = nullptr;
    int32_t* bleaf = nullptr;
    auto free_scratch = [&]() {
        dfree(bk, h->st);
        dfree(br, h->st);
        dfree(bleaf, h->st);
        if (owned) cudaFreeAsync(owned, h->st);
        owned = nullptr;
    };
    auto scratch_guard = at_exit(free_scratch);
    // NEXT-2 fast path (incr.cu): a small batch that keeps the canonical topology is
    // applied by position shifts and a box refit instead of the full rebuild (a
    // single-leaf tree is refused by the check itself).  Its check needs the sorted
    // batch, so small batches sort before the one sync; larger ones sort after it
    // (measured: allocating the batch-sort scratch ahead of the sync makes the stream-
    // ordered pool grow instead of reusing memory in the 10^6-point C5 insert).
    const bool try_fast = incr_enabled() && h->n > 1 && m <= kIncrMaxBatch;
    auto sort_batch = [&]() -> int {
        ZD_CUDA(dalloc(&bk, m, h->st));
        ZD_CUDA(dalloc(&br, m, h->st));
        rec(h, 2);
        return sort_into(h, (const int32_t*)db, m, (uint32_t)first, bk, br);
    };
    if (try_fast) {
        if ((rc = sort_batch())) return rc;
        ZD_CUDA(dalloc(&bleaf, m, h->st));
        KnnArgs t{};
        t.nodes = h->tb.nodes; t.split_bit = h->tb.split_bit; t.d_meta = h->d_small; t.leaf_start = h->tb.leaf_start;
        incr_locate(h->dim, bk, m, t, h->keys, h->leaf_max, bleaf, d_invalid(h) + 1, h->st);
        ZD_CHECK_LAUNCH("incr_locate");
    }
    ZD_CUDA(cudaMemcpyAsync(h->h_small, h->d_small, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, h->st));
    ZD_CUDA(cudaStreamSynchronize(h->st));   // the one sync
    if (h->h_small[4]) return fail(ZD_ERANGE, "zd_insert: coordinate outside the universe box (tree unchanged)");
    if (!try_fast && (rc = sort_batch())) return rc;
    h->n_internal = h->h_small[0];
    h->n_leaves = h->n_internal + 1;
    h->root = h->h_small[1];
    h->host_meta_valid = true;
    const bool fast = try_fast && !h->h_small[5];
    h->poisoned = true;   // cleared when the update completes
    rec(h, 3);
    // growth hands back the old primary arrays as the merge source (no copy)
    uint64_t* src_k = h->keys;
    int4* src_r = h->recs;
    uint64_t* old_k = nullptr;
    int4* old_r = nullptr;
    if ((rc = ensure_id_cap(h, first + m))) return rc;
    if ((rc = ensure_point_cap(h, h->n + m, &old_k, &old_r, fast))) return rc;
    if (old_k) { src_k = old_k; src_r = old_r; }
    // merge into the alternate buffers (K8), then swap
    merge_sorted(src_k, src_r, h->n, bk, br, m, h->keys2, h->recs2, h->st);
    ZD_CHECK_LAUNCH("merge_sorted");
    std::swap(h->keys, h->keys2);
    std::swap(h->recs, h->recs2);
    dfree(old_k, h->st);
    dfree(old_r, h->st);
    if (fast) {
        incr_apply(h->dim, h->n_internal, bleaf, br, m, h->tb.leaf_start, h->tb.pt_leaf, h->tb.nodes, h->tb.range,
                   h->tb.pos_range, h->tb.leaf_parent, h->st);
        ZD_CHECK_LAUNCH("incr_apply");
        h->fast_inserts += 1;
    }
    free_scratch();
    set_alive_range(h->alive, first, m, h->st);
    h->n += m;
    h->n_next += m;
    if (!h->rows_identity) h->rows_dirty = true;
    if ((rc = ensure_rows(h))) return rc;   // zd_knn reads the row map without refreshing it
    rec(h, 4);
    if (fast) {
        if (h->timing) ZD_CUDA(cudaEventRecord(h->ev[6], h->st));   // no topology / box phase
    } else if ((rc = topology(h))) {
        return rc;
    }
    rec(h, 5);
    h->poisoned = false;
    if (h->timing) {
        ZD_CUDA(cudaEventSynchronize(h->ev[5]));
        elapsed(h, PH_VALID, 0, 1);
        elapsed(h, PH_SORT, 2, 3);
        elapsed(h, PH_MERGE, 3, 4);
        elapsed(h, PH_TOPO, 4, 6);
        elapsed(h, PH_BBOX, 6, 5);
    }
    return first;
}

int64_t zd_delete(zd_tree* h, const int32_t* ids, int64_t m) {
    Nvtx range("zd_delete");
    clear_err();
    if (int e = check_handle(h)) return e;
    if (m < 0) return fail(ZD_EINVAL, "zd_delete: m < 0");
    if (m == 0 || h->n == 0) return 0;
    if (!ids) return fail(ZD_EINVAL, "zd_delete: ids is NULL");
    int rc;
    const void* di = nullptr;
    void* owned = nullptr;
    if ((rc = stage_in(h, ids, (size_t)m * sizeof(int32_t), &di, &owned))) return rc;
    rec(h, 0);
    ZD_CUDA(cudaMemsetAsync(d_count(h), 0, sizeof(unsigned long long), h->st));
    mark_deleted(h->alive, h->n_next, (const int32_t*)di, m, d_count(h), h->st);
    compact_alive(h->alive, h->keys, h->recs, h->n, h->keys2, h->recs2, h->tb.block_cnt, h->st);
    ZD_CHECK_LAUNCH("delete");
    if (owned) cudaFreeAsync(owned, h->st);
    // NEXT-2 delete fast path (incr.cu): checked on the device before the one sync,
    // which reads the deleted count, the check's verdict and the node meta together
    int32_t* del_before = nullptr;
    uint32_t* dscratch = nullptr;
    auto scratch_guard = at_exit([&]() { dfree(del_before, h->st); dfree(dscratch, h->st); });
    const bool try_fast = incr_enabled() && m <= kIncrMaxBatch && h->n > 1;
    const int64_t ncap = h->ncap, nblk_cap = (ncap + 1 + 255) / 256;
    if (try_fast) {
        ZD_CUDA(dalloc(&del_before, ncap + 2, h->st));
        ZD_CUDA(dalloc(&dscratch, 2 * ncap + nblk_cap + 2, h->st));   // mark [ncap] | arrived [ncap] | bsum
        ZD_CUDA(cudaMemsetAsync(d_invalid(h) + 1, 0, sizeof(int), h->st));
        decr_check(ncap, h->d_small, h->recs, h->tb.leaf_start, h->alive, h->tb.range, h->leaf_max, del_before,
                   dscratch + 2 * ncap, d_invalid(h) + 1, h->st);
        ZD_CHECK_LAUNCH("decr_check");
    }
    ZD_CUDA(cudaMemcpyAsync(h->h_small, h->d_small, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, h->st));
    rec(h, 1);
    ZD_CUDA(cudaStreamSynchronize(h->st));   // the one sync
    h->n_internal = h->h_small[0];
    h->n_leaves = h->n_internal + 1;
    h->root = h->h_small[1];
    h->host_meta_valid = true;
    unsigned long long cnt;
    std::memcpy(&cnt, h->h_small + 6, sizeof(cnt));
    if (cnt == 0) return 0;
    const bool fast = try_fast && !h->h_small[5];
    h->poisoned = true;   // cleared when the update completes
    std::swap(h->keys, h->keys2);
    std::swap(h->recs, h->recs2);
    h->n -= (int64_t)cnt;
    h->rows_identity = false;
    h->rows_dirty = true;
    if ((rc = ensure_rows(h))) return rc;   // zd_knn reads the row map without refreshing it
    rec(h, 2);
    if (fast) {
        const int64_t nb = h->n_internal;
        ZD_CUDA(cudaMemsetAsync(dscratch, 0, 2 * nb * sizeof(uint32_t), h->st));   // mark | arrived
        decr_apply(h->dim, nb, del_before, h->tb.leaf_start, h->tb.pt_leaf, h->tb.nodes, h->tb.range, h->tb.pos_range,
                   h->tb.leaf_parent, h->recs, dscratch, dscratch + nb, h->st);
        ZD_CHECK_LAUNCH("decr_apply");
        h->fast_deletes += 1;
        if (h->timing) ZD_CUDA(cudaEventRecord(h->ev[6], h->st));
    } else if ((rc = topology(h))) {
        return rc;
    }
    rec(h, 3);
    h->poisoned = false;
    if (h->timing) {
        ZD_CUDA(cudaEventSynchronize(h->ev[3]));
        elapsed(h, PH_MERGE, 0, 1);
        elapsed(h, PH_TOPO, 2, 6);
        elapsed(h, PH_BBOX, 6, 3);
    }
    return (int64_t)cnt;
}

int zd_live_ids(const zd_tree* hc, int32_t* out) {
    clear_err();
    zd_tree* h = const_cast<zd_tree*>(hc);
    if (int e = check_handle(h)) return e;
    if (!out && h->n > 0) return fail(ZD_EINVAL, "NULL argument");
    if (h->n == 0) return ZD_OK;
    int rc;
    if (h->rows_identity) {
        // ids 0..n-1 are all alive: identity
        rank_alive(h->alive, h->n_next, h->row_of_id, h->live_ids, h->rank_cnt, h->st);
        ZD_CHECK_LAUNCH("rank_alive");
    } else if ((rc = ensure_rows(h))) {
        return rc;
    }
    ZD_CUDA(cudaMemcpyAsync(out, h->live_ids, h->n * sizeof(int32_t), cudaMemcpyDefault, h->st));
    ZD_CUDA(cudaStreamSynchronize(h->st));
    return ZD_OK;
}

int zd_get_info(const zd_tree* hc, zd_info* out) {
    zd_tree* h = const_cast<zd_tree*>(hc);
    if (!h || !out) return fail(ZD_EINVAL, "NULL argument");
    int rc = refresh_host_meta(h);
    if (rc) return rc;
    out->dim = h->dim;
    out->leaf_max = h->leaf_max;
    out->n = h->n;
    out->n_next = h->n_next;
    out->n_leaves = h->n_leaves;
    out->n_internal = h->n_internal;
    out->root = h->root;
    out->node_words = h->dim == 2 ? 12 : 16;
    for (int a = 0; a < 3; ++a) out->shift[a] = h->shift[a];
    out->fast_inserts = h->fast_inserts;
    out->fast_deletes = h->fast_deletes;
    out->sort_fallbacks = h->trunc_fallbacks;
    return ZD_OK;
}

int zd_export(const zd_tree* hc, uint64_t* keys, int32_t* recs, int32_t* leaf_start, int32_t* leaf_parent,
              int32_t* nodes) {
    zd_tree* h = const_cast<zd_tree*>(hc);
    if (int e = check_handle(h)) return e;
    int rc = refresh_host_meta(h);
    if (rc) return rc;
    const cudaMemcpyKind K = cudaMemcpyDefault;
    if (keys && h->n) ZD_CUDA(cudaMemcpyAsync(keys, h->keys, h->n * sizeof(uint64_t), K, h->st));
    if (recs && h->n) ZD_CUDA(cudaMemcpyAsync(recs, h->recs, h->n * sizeof(int4), K, h->st));
    if (leaf_start) ZD_CUDA(cudaMemcpyAsync(leaf_start, h->tb.leaf_start, (h->n_leaves + 1) * sizeof(int32_t), K, h->st));
    if (leaf_parent) ZD_CUDA(cudaMemcpyAsync(leaf_parent, h->tb.leaf_parent, h->n_leaves * sizeof(int32_t), K, h->st));
    if (nodes && h->n_internal) {
        const size_t bytes = (size_t)h->n_internal * (4 * h->dim + 4) * sizeof(int32_t);
        int32_t* tmp = nullptr;
        ZD_CUDA(pool_alloc((void**)&tmp, bytes, h->st));
        export_nodes(h->dim, h->tb.nodes, h->tb.split_bit, h->n_internal, tmp, h->st);
        ZD_CHECK_LAUNCH("export_nodes");
        ZD_CUDA(cudaMemcpyAsync(nodes, tmp, bytes, K, h->st));
        ZD_CUDA(cudaFreeAsync(tmp, h->st));
    }
    ZD_CUDA(cudaStreamSynchronize(h->st));
    return ZD_OK;
}

}  // extern "C"
