// internal.h — host-side launch interface between the CUDA translation units.
#pragma once

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

namespace zd {

// One-time setup per CUDA device (devices 0..63), safe under concurrent callers: the
// per-device flag is published with release order after f() ran, under a mutex.
struct PerDeviceOnce {
    std::atomic<uint64_t> done{0};
    std::mutex mu;
    template <class F>
    void run(F&& f) {
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t bit = 1ull << (dev & 63);
        if (done.load(std::memory_order_acquire) & bit) return;
        std::lock_guard<std::mutex> g(mu);
        if (done.load(std::memory_order_relaxed) & bit) return;
        f(dev);
        done.fetch_or(bit, std::memory_order_release);
    }
};

// Stream-ordered allocations come from a private memory pool per device (not the
// device's default pool, which other code in the process may use), with the release
// threshold raised so repeated builds reuse memory; zd_trim() hands it back.
cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t st);

// process-wide count of kernel launches issued by this library (zd_kernel_launches)
void count_launch(int k = 1);

// ---------------------------------------------------------------- sort (sort.cu)
// One-sweep LSD radix sort of (Morton key, id): 8 passes x 8-bit digits, one
// up-front histogram of all 8 digits, decoupled look-back per pass.
struct SortScratch {
    uint64_t* k[2];        // ping-pong keys   [cap]
    uint32_t* v[2];        // ping-pong ids    [cap]
    uint32_t* zero_block;  // hist[8*256] | counters[8] | status[8*tiles*256] (memset as one block)
    uint32_t* offs;        // [8*256] exclusive digit offsets
    size_t zero_words;
};
size_t sort_tiles(int64_t n);
size_t sort_zero_words(int64_t n);
// Encode pts (int32 [n][dim]) and sort; ids = id_base + i.  Writes sorted keys
// and records int4(x, y, z|0, id).  Sets *d_invalid != 0 if a coordinate is out of
// the universe box.
// shift2: the random shift (int32 [dim]) added after the range check, or NULL (2D:
// 62-bit keys; 3D: keys of the shifted coordinates' levels 21..1, records gathered
// from the input points).
// d_trunc_fail != NULL: the truncated sort (5 passes + a rank fixup of equal-prefix
// runs); *d_trunc_fail is set if a run was too long, and the caller must redo the sort
// with d_trunc_fail == NULL (all 8 passes) before using the output.  approx: order
// by key bits 24..63 only (5 passes, no fixup) — for query batches, whose order only
// serves locality.
void sort_points(int dim, const int32_t* pts, int64_t n, uint32_t id_base, uint64_t* keys_out,
                 int4* recs_out, const SortScratch& s, int* d_invalid, cudaStream_t st,
                 const int32_t* shift2 = nullptr, int* d_trunc_fail = nullptr, bool approx = false);
// The same order for n <= kSmallSort keys in one single-block launch (no scratch).
constexpr int kSmallSort = 256;
void sort_points_small(int dim, const int32_t* pts, int64_t n, uint32_t id_base, uint64_t* keys_out, int4* recs_out,
                       int* d_invalid, cudaStream_t st, const int32_t* shift2 = nullptr);

// ---------------------------------------------------------------- tree (tree.cu)
struct TreeBufs {
    int32_t* pt_leaf;      // [cap]   leaf of each sorted position
    int32_t* leaf_start;   // [cap+2]
    int32_t* leaf_parent;  // [cap+1]
    int32_t* split_bit;    // [cap]   per internal node (in-order)
    void* nodes;           // [cap]   Node<dim>
    uint32_t* visit;       // [cap]   bottom-up arrival counters
    int32_t* range;        // [2*cap] bottom-up leaf-range scratch
    int2* pos_range;       // [cap]   sorted point range [x, y) of internal node i
    uint8_t* flags;        // [cap]   big-pair flags
    uint32_t* block_cnt;   // [tree_blocks(cap)+1]
    int32_t* d_meta;       // [4]: nb (internal count), root ref
};
size_t tree_blocks(int64_t n);
// Canonical topology (K4) + bottom-up boxes (K5) over sorted keys/records.
void build_topology(int dim, const uint64_t* keys, const int4* recs, int64_t n, int leaf_max,
                    const TreeBufs& t, cudaStream_t st, cudaEvent_t ev_mid);
// The same in two halves (n >= 2): big-pair flags + block scan (the internal-node
// count lands in block_cnt[tree_blocks(n)]), then compaction + bottom-up boxes.
void topology_flags(const uint64_t* keys, int64_t n, int leaf_max, const TreeBufs& t, cudaStream_t st);
void topology_finish(int dim, const uint64_t* keys, const int4* recs, int64_t n, const TreeBufs& t,
                     cudaStream_t st, cudaEvent_t ev_mid);
// Internal nodes in the documented zd_export layout (leaf children as ~leaf index,
// split bit last) into out int32 [nb][4*dim+4].
void export_nodes(int dim, const void* nodes, const int32_t* split_bit, int64_t nb, int32_t* out, cudaStream_t st);

// ---------------------------------------------------------------- knn (knn.cu)
struct KnnArgs {
    int dim, k;
    int64_t n;                   // live points
    const int4* recs;
    const int32_t* pt_leaf;
    const int32_t* leaf_start;
    const int32_t* leaf_parent;
    const void* nodes;
    const int32_t* node_range;   // [2*n_internal]: leaves [L, R] under internal node i
    const int2* pos_range;       // [n_internal]: sorted point range of internal node i
    const int32_t* split_bit;    // [n_internal]
    const int32_t* d_meta;       // root ref at [1]
    const int32_t* row_of_id;    // NULL: row = id
    int32_t* out_idx;
    int64_t* out_d2;
    int32_t* hard_list;          // [hard_cap] scratch for deferred packets (NULL: none)
    int32_t* hard_count;         // [0] deferred packets, [1] persistent packet counter: zeroed by the caller
    int hard_cap;
    int defer_all;               // testing: every packet goes to the second pass
    int root_based;              // ablation: root-based search
    int warp;                    // the warp-per-query kernel (knn_warp.cu) for any k
    int64_t q_lo, q_hi;          // all-points: query the live points at sorted positions [q_lo, q_hi)
};
constexpr int kPacketKMax = 32;   // largest k of the packet kernel; above: knn_warp
// Large-k path (knn_warp.cu): one warp per query over Morton-ordered queries.
void knn_warp(const KnnArgs& a, const int4* qrecs, const int32_t* qleaf, int64_t nq, bool ext, cudaStream_t st);
// NEXT-2 insert fast path (incr.cu): leaf of each sorted batch key by its bits, *bad set
// if a key leaves its leaf's cell or a leaf would exceed leaf_max; then the in-place
// position shifts and box refit for a batch that keeps the topology.
void incr_locate(int dim, const uint64_t* bkeys, int64_t m, const KnnArgs& t, const uint64_t* keys, int leaf_max,
                 int32_t* bleaf, int* bad, cudaStream_t st);
void incr_apply(int dim, int64_t nb, const int32_t* bleaf, const int4* brecs, int64_t m, int32_t* leaf_start,
                int32_t* pt_leaf, void* nodes, const int32_t* range, int2* pos_range, const int32_t* leaf_parent,
                cudaStream_t st);
// Delete fast path: dead records per leaf (old arrays + alive bitset) scanned into
// del_before [nleaves+1] (bsum: block scratch), *bad if a leaf empties, an internal
// node drops to <= leaf_max points or the tree is a single leaf; then the position
// shifts and dirty-path box refit (mark, arrived: zeroed node-sized scratch).  The
// check is launched over the node capacity nb_cap and reads the node count from the
// device meta (meta[0] internal nodes, meta[1] root): no host sync before it.
int decr_check(int64_t nb_cap, const int32_t* meta, const int4* recs_old, const int32_t* leaf_start,
               const uint32_t* alive, const int32_t* range, int leaf_max, int32_t* del_before, uint32_t* bsum, int* bad,
               cudaStream_t st);
void decr_apply(int dim, int64_t nb, const int32_t* del_before, int32_t* leaf_start, int32_t* pt_leaf, void* nodes,
                const int32_t* range, int2* pos_range, const int32_t* leaf_parent, const int4* recs_new, uint32_t* mark,
                uint32_t* arrived, cudaStream_t st);
// Work counters of the packet k-NN kernel (only in a -DZD_KNN_STATS build).
enum { ZS_PACKETS = 0, ZS_QUERIES, ZS_NODES, ZS_POPS, ZS_ASCENTS, ZS_SPANS, ZS_PASSES, ZS_CAND, ZS_HITS,
       ZS_ROUNDS, ZS_COMPACT, ZS_SURV, ZS_SURV_MAX, ZS_CYCLES, ZS_MAXPKT, ZS_DEFERRED, ZS_HIST0, ZS_INS = ZS_HIST0 + 32,
       ZS_SEED_HITS, ZS_SEED_INS, ZS_SEED_ROUNDS, ZS_LANE_COMPACT, ZS_NEED_PAIRS, ZS_RAW, ZD_NSTATS };
int knn_stats(unsigned long long* out, int n, int reset);
void knn_all(const KnnArgs& a, cudaStream_t st);
// External queries, already Morton-sorted (qkeys, qrecs with w = query index):
// bit-based leaf location into qleaf [m], then the packet search (row = query index).
void knn_queries(const KnnArgs& a, const uint64_t* qkeys, const int4* qrecs, int32_t* qleaf, int64_t m,
                 cudaStream_t st);

// ---------------------------------------------------------------- updates (update.cu)
void validate_points(int dim, const int32_t* pts, int64_t m, int* d_invalid, cudaStream_t st);
// Merge sorted (ka, ra)[n] with sorted (kb, rb)[m] by key (a before b on equal keys).
void merge_sorted(const uint64_t* ka, const int4* ra, int64_t n, const uint64_t* kb, const int4* rb,
                  int64_t m, uint64_t* ko, int4* ro, cudaStream_t st);
// alive bitset ops
void set_alive_range(uint32_t* alive, int64_t first, int64_t count, cudaStream_t st);
void mark_deleted(uint32_t* alive, int64_t id_cap, const int32_t* ids, int64_t m,
                  unsigned long long* d_count, cudaStream_t st);
// keep sorted positions whose id is alive; returns nothing (count known from d_count)
void compact_alive(const uint32_t* alive, const uint64_t* ki, const int4* ri, int64_t n,
                   uint64_t* ko, int4* ro, uint32_t* block_cnt, cudaStream_t st);
size_t compact_blocks(int64_t n);
// row_of_id[id] = rank of id among alive ids (for ids < id_cap); live_ids[rank] = id
void rank_alive(const uint32_t* alive, int64_t id_cap, int32_t* row_of_id, int32_t* live_ids,
                uint32_t* block_cnt, cudaStream_t st);
size_t rank_blocks(int64_t id_cap);

}  // namespace zd
