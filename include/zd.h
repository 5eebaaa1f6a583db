/*
 * zd.h — C ABI of the B200-native zd-tree hot path.
 *
 * The zd-tree is a kd-tree whose splits follow the Morton (z-order) bit
 * interleaving (§2 "Data structure"; Blelloch & Dobson,
 * arXiv 2111.04182).  This library implements, as hand-written sm_100a CUDA
 * kernels on one GPU:
 *   zd_build  — Morton encode + radix sort of (key, id) + tree cut at the highest
 *               differing bit + bottom-up bounding boxes  (§2
 *               "Construction"; Alg. 1 buildTree P:255-275; empty cuts P:463)
 *   zd_knn    — all-points exact k-NN graph, leaf-based searchUp/searchDown
 *               (Alg. 3, Alg. 2, "leaf-based" P:248), or
 *               external queries located by their Morton bits ("bit-based" P:248)
 *   zd_insert — batch insert (Alg. 4 batchInsert P:354-377)
 *   zd_delete — batch delete ("almost identical")
 *
 * Domain (fixed universe box; SURVEY.md §8(c) reading 5):
 *   dim = 2: int32 coordinates with 0 <= c < 2^30  (60-bit Morton keys)
 *   dim = 3: int32 coordinates with 0 <= c < 2^21  (63-bit Morton keys)
 * Distances are exact int64 squared Euclidean distances.
 *
 * Result semantics (SURVEY §8(c) "Result definition"; readings 13-15, 21):
 *   row r of an all-points query belongs to the r-th smallest live id; it holds
 *   the first min(k, L-1) pairs of {(d2(q, p_j), j) : j live, j != id(q)} in
 *   lexicographic (d2, id) order, padded with (-1, INT64_MAX).  The answer is
 *   unique, so GPU and oracle rows are compared bit-exactly.
 *
 * Pointers: every array argument may be a CUDA device pointer OR a host pointer
 * (pageable or pinned); the library detects which with
 * cudaPointerGetAttributes and stages host arrays through device memory itself
 * (host outputs are complete when the call returns).  Arrays are dense,
 * row-major, little-endian.  The library copies what it needs from inputs, so the
 * caller keeps ownership of every buffer it passes and may free it after return.
 *
 * Streams: all work runs on the handle's stream (zd_build_ex opts / zd_set_stream;
 * default: the legacy default stream).  zd_build, zd_insert and zd_delete
 * synchronize that stream once (to read a validation flag, the tree's node count or
 * the deleted count); only trees above 2^25 points, whose node buffers are sized
 * from the node count, take one more sync per topology rebuild.  zd_knn with device
 * outputs is asynchronous on the stream.
 *
 * Errors: functions returning int/int64 return a negative ZD_E* code on failure;
 * functions returning pointers return NULL.  zd_last_error() gives a
 * thread-local message for the most recent failure on the calling thread.
 * Validation happens before any mutation: a failed insert leaves the tree
 * unchanged (S:383 all-or-nothing).
 *
 * Concurrency: zd_knn may be called concurrently on one handle from several host
 * threads ("queries can be conducted in parallel"): it only reads the handle
 * (the row map of the all-points output is refreshed by zd_insert / zd_delete),
 * allocates its scratch per call and times itself with events of its own; device
 * work of concurrent calls is ordered on the handle's stream.  zd_insert /
 * zd_delete / zd_set_stream / zd_set_timing / zd_free need exclusive access.
 */
#ifndef ZD_H
#define ZD_H

#include <stdint.h>

#if defined(__GNUC__)
#define ZD_API __attribute__((visibility("default")))
#else
#define ZD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct zd_tree zd_tree;  /* opaque; owns all device memory it allocates */

enum {
    ZD_OK = 0,
    ZD_EINVAL = -1,   /* bad argument (dim, n, k, m, NULL handle, ...) */
    ZD_ERANGE = -2,   /* a coordinate outside the universe box */
    ZD_ENOMEM = -3,   /* device allocation failed */
    ZD_ECUDA = -4     /* any other CUDA runtime error */
};

#define ZD_K_MAX 128       /* largest k served by zd_knn (k > 32: warp-per-query path) */
#define ZD_LEAF_MAX_MAX 32 /* largest leaf size accepted by zd_build_ex */

typedef struct zd_opts {
    void *stream;   /* cudaStream_t for all work; NULL = legacy default stream */
    int leaf_max;   /* leaf size bound (reading 1: leaf iff size <= leaf_max or all
                       keys equal); 0 = default 16; valid 1..ZD_LEAF_MAX_MAX */
    int timing;     /* nonzero: record per-phase device times (zd_get_timing) */
    /* Random shift (§2, "select a random shift ... kept throughout"; Lemma 2.2
     * P:450): shift_set != 0 adds shift[a] to axis a of every point — build points,
     * inserted batches and external queries alike — after the range check and before
     * encoding.  2D: shift[a] in [0, 2^30), shifted coordinates of 31 bits, 62-bit
     * keys.  3D: shift[a] in [0, 2^21), shifted coordinates of 22 bits; the key
     * interleaves their levels 21..1 (63 bits: the Morton order of the shifted grid at
     * cell size 2, DESIGN reading R31) while records keep the exact shifted
     * coordinates.  Other shifts return ZD_EINVAL.  Distances, neighbour ids and rows
     * are unchanged (a translation); the tree is the canonical tree of the shifted
     * points and zd_export reports shifted keys and coordinates.  The caller draws the
     * shift. */
    int shift_set;
    int32_t shift[3];
} zd_opts;

/* Build a zd-tree over n points (int32 [n][dim]); point i gets id i.
 * n = 0 is valid (single empty leaf).  Returns NULL on error: dim not in {2,3},
 * n < 0 or n >= 2^30 (ZD_EINVAL: one radix sort holds < 2^30 keys), a coordinate
 * outside the box (ZD_ERANGE),
 * allocation/CUDA failure.  Cite: Alg. 1 P:255-275. */
ZD_API zd_tree *zd_build(const int32_t *points, int64_t n, int dim);
ZD_API zd_tree *zd_build_ex(const int32_t *points, int64_t n, int dim, const zd_opts *opts);

/* Exact k nearest neighbours.
 *   queries == NULL: all-points k-NN graph over the live points (leaf-based,
 *     P:248); m must equal zd_size(h); row r = r-th smallest live id (zd_live_ids);
 *     the query point itself is excluded by id.
 *   queries != NULL: m external query points int32 [m][dim] inside the box
 *     (bit-based; "dynamic queries" P:183); row j = query j; nothing excluded.
 * out_idx: int32 [m][k] neighbour ids; out_dist2: int64 [m][k] squared distances.
 * 1 <= k <= ZD_K_MAX.  Returns ZD_OK or a negative code (ZD_EINVAL for bad k/m,
 * ZD_ERANGE for an out-of-box query). */
ZD_API int zd_knn(zd_tree *h, const int32_t *queries, int64_t m, int k,
           int32_t *out_idx, int64_t *out_dist2);

/* zd_knn with options.  flags: 0 = zd_knn (leaf-based search: every query
 * starts at its own leaf and ascends, Alg. 3); ZD_KNN_ROOT_BASED = the
 * root-based variant (Alg. 2 from the root with an empty neighbour list), kept
 * as an ablation — the answer is identical, the work differs (the paper's Fig. 2).
 * ZD_KNN_WARP = run the large-k kernel (one warp per query, warp-shared top-k buffer
 * with radix selection; P:543's large-k container) for any k; it
 * always serves k > 32.  Flags combine.  Unknown flags -> ZD_EINVAL. */
#define ZD_KNN_ROOT_BASED 1
#define ZD_KNN_WARP 2
ZD_API int zd_knn_ex(zd_tree *h, const int32_t *queries, int64_t m, int k,
              int32_t *out_idx, int64_t *out_dist2, int flags);

/* All-points k-NN restricted to the live points at sorted (Morton) positions
 * [pos_lo, pos_hi) — one shard of the parallel-for over queries (
 * SURVEY §8(e) item 1): every GPU holding a replica of the tree answers a contiguous
 * Morton range, so together they produce the all-points output with no exchange.
 * Writes only those points' rows of the full row-major outputs int32 / int64
 * [zd_size(h)][k] (row = rank of the point's id among the live ids, as in zd_knn);
 * other rows are untouched.  0 <= pos_lo <= pos_hi <= zd_size(h); the outputs must be
 * device arrays (ZD_EINVAL otherwise); flags as zd_knn_ex.  Asynchronous. */
ZD_API int zd_knn_range(zd_tree *h, int64_t pos_lo, int64_t pos_hi, int k,
                        int32_t *out_idx, int64_t *out_dist2, int flags);

/* Insert m points (int32 [m][dim]); they get ids first, first+1, ... where
 * first = the next unused id (ids are never reused, reading 20); 0 <= m < 2^30.
 * Returns first (>= 0) or a negative code; on a validation error (ZD_EINVAL,
 * ZD_ERANGE) the tree is unchanged; a CUDA failure during the update leaves the handle
 * unusable (later calls return ZD_ECUDA; free it).  The tree after the
 * call is the canonical zd-tree of the live multiset (reading 17).  Alg. 4
 * P:354-377. */
ZD_API int64_t zd_insert(zd_tree *h, const int32_t *batch, int64_t m);

/* Delete the points with the given ids (int32 [m]).  Absent, already-deleted and
 * duplicate ids are skipped.  Returns the number of points deleted, or a
 * negative code.  P:253. */
ZD_API int64_t zd_delete(zd_tree *h, const int32_t *ids, int64_t m);

/* Number of live points (>= 0), or ZD_EINVAL for a NULL handle. */
ZD_API int64_t zd_size(const zd_tree *h);

/* Write the live ids in ascending order (int32 [zd_size(h)]) = the row order of
 * the all-points output (reading 21).  Synchronous. */
ZD_API int zd_live_ids(const zd_tree *h, int32_t *out);

/* Make all later work on h run on the given cudaStream_t (NULL = legacy default). */
ZD_API int zd_set_stream(zd_tree *h, void *cuda_stream);

/* Free the handle and all its device memory (NULL is a no-op).  The memory goes back
 * to the library's private stream-ordered pool of the device (cached for the next
 * build); zd_trim releases it. */
ZD_API void zd_free(zd_tree *h);

/* Release the memory cached in the library's pool on the current device back to the
 * driver (cudaMemPoolTrimTo 0 after a device synchronize); live handles keep theirs.
 * Returns ZD_OK or ZD_ECUDA. */
ZD_API int zd_trim(void);

/* Thread-local message for the last error on this thread ("" if none). */
ZD_API const char *zd_last_error(void);

/* Thread-local ZD_E* code of the last error on this thread (ZD_OK if none). */
ZD_API int zd_last_error_code(void);

/* ---- introspection (structural-parity tests and benchmarking) ---------- */

typedef struct zd_info {
    int dim;
    int leaf_max;
    int64_t n;            /* live points */
    int64_t n_next;       /* next id to be assigned */
    int64_t n_leaves;     /* leaves of the canonical tree (= n_internal + 1) */
    int64_t n_internal;   /* internal nodes */
    int32_t root;         /* root reference: >= 0 internal node, < 0 leaf ~ref */
    int32_t node_words;   /* int32 words per exported internal node */
    int32_t shift[3];     /* zd_opts.shift as applied (zeros: none) */
    int64_t fast_inserts; /* inserts applied without a topology rebuild (NEXT-2 fast
                             path: the batch kept the canonical topology; ZD_INCR=0
                             in the environment disables it) */
    int64_t fast_deletes; /* deletes applied without a topology rebuild (no leaf
                             emptied, every internal node kept > leaf_max points) */
    int64_t sort_fallbacks; /* builds (n >= 2^20) whose truncated sort — 5 radix passes
                             over key bits 24..63, then each run of equal 40-bit prefixes
                             ranked by (key, id) — met a run longer than 64 and was
                             redone with all 8 passes (degenerate, clustered inputs) */
} zd_info;

ZD_API int zd_get_info(const zd_tree *h, zd_info *out);

/* Copy the tree out (synchronous; any pointer may be NULL to skip it):
 *   keys        uint64 [n]      sorted Morton keys (by key, then id)
 *   recs        int32 [n][4]    (x, y, z-or-0, id) in the same order
 *   leaf_start  int32 [n_leaves+1]  leaf l covers sorted positions
 *                                   [leaf_start[l], leaf_start[l+1])
 *   leaf_parent int32 [n_leaves]    internal node index, -1 for a root leaf
 *   nodes       int32 [n_internal][node_words]: internal node i (in-order: it
 *               separates leaf i from leaf i+1) = left-child box (lo[dim], hi[dim]),
 *               right-child box (lo[dim], hi[dim]), left ref, right ref, parent,
 *               split bit.  A ref >= 0 is an internal node, a ref < 0 is leaf ~ref. */
ZD_API int zd_export(const zd_tree *h, uint64_t *keys, int32_t *recs, int32_t *leaf_start,
              int32_t *leaf_parent, int32_t *nodes);

/* Per-phase device times (ms, CUDA events on the handle's stream) of the most
 * recent zd_build / zd_insert / zd_delete / zd_knn call, when enabled by
 * zd_set_timing(h, 1).  Phases: 0 encode+sort, 1 topology, 2 bbox (bottom-up),
 * 3 merge/compaction, 4 knn, 5 validation.  Fills min(nphase, 6) entries and
 * returns the number filled.  Timing adds event records but no extra syncs
 * beyond the ones each call already makes (zd_knn syncs when timing is on). */
ZD_API int zd_set_timing(zd_tree *h, int enable);
/* Process-wide number of CUDA kernels this library has launched so far. */
ZD_API int64_t zd_kernel_launches(void);
ZD_API int zd_get_timing(const zd_tree *h, float *ms, int nphase);

/* Work counters accumulated by the k-NN kernel since the last reset, for profiling
 * builds only (compiled with -DZD_KNN_STATS; a normal build returns ZD_EINVAL).
 * Order: packets, queries, internal nodes visited, stack pops, ascents, scanned
 * spans, uniform passes, candidates tested (per warp), hits (sum over lanes),
 * hit rounds (max over lanes per pass), compactions, final survivors (sum over
 * lanes), final survivors (max over lanes per packet).  Fills min(n, 13) int64
 * entries, returns the number filled; reset != 0 zeroes the counters after reading. */
ZD_API int zd_knn_stats(int64_t *out, int n, int reset);

#ifdef __cplusplus
}
#endif

#endif /* ZD_H */
