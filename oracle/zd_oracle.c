/*
 * zd_oracle.c — plain, slow, obviously-correct CPU oracle for the zd-tree hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2111_04182_b200/) never includes, links or calls it, and this file
 * includes nothing from the product (no shared headers, helpers or tables).
 *
 * Citations: "P:n" = line n of PAPER.md (Blelloch & Dobson, arXiv 2111.04182);
 * "S:n" = line n of SPEC.md.  Readings of ambiguous passages are numbered as in
 * SURVEY.md §8(c) and listed in DESIGN.md "Readings".
 *
 * What it computes:
 *   keys   — Morton interleave by a scalar bit loop (§1.1; S:49 dim 0 most
 *            significant within a bit group).  Deliberately NOT a magic-number spread.
 *            B = 30 (2D) / 21 (3D) bits per axis; 31 in 2D when the caller applies
 *            the random shift of P:235 (orc_build_bits; the Python Tree(shift=)).
 *   sort   — qsort by (key, id) (§2).
 *   build  — recursive Alg. 1 buildTree/splitUsingBit with empty
 *            cuts skipped: leaf iff size <= leaf_max or all keys equal
 *            (readings 1-3); otherwise cut at the highest differing bit of
 *            key[lo]^key[hi-1] and split at the first index whose bit is 1
 *            (binary search).  Tight per-axis bboxes (reading 7).
 *   query  — Alg. 3 searchUp calling Alg. 2 searchDown,
 *            k-best set ordered by (d^2, id) (readings 8, 9, 13, 14), self
 *            excluded by id, rows padded with (-1, INT64_MAX) (reading 15).
 *            Also: root-based Alg. 2 from the root and bit-based external
 *            queries for cross-variant checks.
 *   brute  — O(n) scan per query: the plain definition of the answer.
 */
#define _GNU_SOURCE
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <sched.h>
#include <unistd.h>

#define ORC_DMAX_INF INT64_MAX

/* ------------------------------------------------------------------ keys */

static int bits_per_axis(int dim) { return dim == 2 ? 30 : 21; }

/* "taking each integer coordinate in binary form, interleaving the
 * coordinates to create one integer per point".  Level l = B-1 .. 0, axis
 * 0 .. dim-1, key = (key << 1) | bit. */
static uint64_t key_levels(const int32_t *c, int dim, int B, int lo) {
    uint64_t key = 0;
    for (int l = B - 1; l >= lo; --l)
        for (int a = 0; a < dim; ++a)
            key = (key << 1) | (uint64_t)(((uint32_t)c[a] >> l) & 1u);
    return key;
}

static uint64_t key_bits(const int32_t *c, int dim, int B) { return key_levels(c, dim, B, 0); }

uint64_t orc_key(const int32_t *c, int dim) { return key_bits(c, dim, bits_per_axis(dim)); }

void orc_keys(const int32_t *pts, int64_t n, int dim, uint64_t *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_key(pts + i * dim, dim);
}

/* Returns 1 iff every coordinate lies in the fixed universe box [0, 2^B). */
int orc_in_box(const int32_t *pts, int64_t n, int dim) {
    int64_t lim = (int64_t)1 << bits_per_axis(dim);
    for (int64_t i = 0; i < n * dim; ++i)
        if (pts[i] < 0 || (int64_t)pts[i] >= lim) return 0;
    return 1;
}

/* ------------------------------------------------------------ geometry */

/* Squared distance from q to the nearest point of box [lo, hi]; 0 inside
 * (withinBox, Alg. 2 caption P:283-284). */
int64_t orc_boxd2(const int32_t *q, const int32_t *lo, const int32_t *hi, int dim) {
    int64_t s = 0;
    for (int a = 0; a < dim; ++a) {
        int64_t d = 0;
        if (q[a] < lo[a]) d = (int64_t)lo[a] - q[a];
        else if (q[a] > hi[a]) d = (int64_t)q[a] - hi[a];
        s += d * d;
    }
    return s;
}

/* Smallest per-axis margin of q inside [lo, hi] (withinBox with negative r,
 * Alg. 3 caption P:323-324).  Negative if q is outside. */
int64_t orc_margin(const int32_t *q, const int32_t *lo, const int32_t *hi, int dim) {
    int64_t m = INT64_MAX;
    for (int a = 0; a < dim; ++a) {
        int64_t l = (int64_t)q[a] - lo[a], h = (int64_t)hi[a] - q[a];
        int64_t t = l < h ? l : h;
        if (t < m) m = t;
    }
    return m;
}

static int64_t dist2(const int32_t *a, const int32_t *b, int dim) {
    int64_t s = 0;
    for (int t = 0; t < dim; ++t) {
        int64_t d = (int64_t)a[t] - b[t];
        s += d * d;
    }
    return s;
}

/* --------------------------------------------------------- k-best set */
/* Sorted ascending by (d^2, id) — reading 14. */
typedef struct {
    int k, cnt;
    int64_t *d;
    int32_t *id;
} nset;

static int pair_less(int64_t d1, int32_t i1, int64_t d2, int32_t i2) {
    return d1 < d2 || (d1 == d2 && i1 < i2);
}

/* distance(p, N, k) of Alg. 2: +inf while |N| < k. */
static int64_t nset_radius(const nset *N) { return N->cnt < N->k ? ORC_DMAX_INF : N->d[N->k - 1]; }

/* insert(N, q, k) (reading 11): keep the k smallest (d^2, id). */
static int nset_insert(nset *N, int64_t d, int32_t id) {
    int pos;
    if (N->cnt < N->k) {
        pos = N->cnt++;
    } else {
        if (!pair_less(d, id, N->d[N->k - 1], N->id[N->k - 1])) return 0;
        pos = N->k - 1;
    }
    while (pos > 0 && pair_less(d, id, N->d[pos - 1], N->id[pos - 1])) {
        N->d[pos] = N->d[pos - 1];
        N->id[pos] = N->id[pos - 1];
        --pos;
    }
    N->d[pos] = d;
    N->id[pos] = id;
    return 1;
}

/* Test hook for the S:264-266 worked examples. */
int orc_nset_demo(int k, const int64_t *d, const int32_t *id, int m, int64_t *out_d, int32_t *out_id) {
    nset N = {k, 0, out_d, out_id};
    for (int i = 0; i < k; ++i) { out_d[i] = ORC_DMAX_INF; out_id[i] = -1; }
    for (int i = 0; i < m; ++i) nset_insert(&N, d[i], id[i]);
    return N.cnt;
}

/* ----------------------------------------------------------------- tree */

typedef struct {
    uint64_t key;
    int32_t id;
    int32_t c[3];
} orc_pt;

typedef struct {
    int64_t lo, hi;     /* range of sorted points [lo, hi) */
    int32_t split;      /* split bit; -1 for a leaf */
    int32_t parent, left, right;
    int32_t bmin[3], bmax[3];
} orc_node;

typedef struct orc_tree {
    int dim, leaf_max;
    int64_t n;
    orc_pt *pts;        /* sorted by (key, id) */
    orc_node *nodes;
    int32_t nnodes, cap, root;
    int32_t *leaf_of;   /* sorted position -> leaf node */
    int64_t *row_of;    /* sorted position -> output row (rank of id among ids) */
    int bits;          /* key bits per axis: levels bits-1 .. lo of every coordinate */
    int lo;            /* lowest level in the key (1 in the 3D random-shift mode, else 0) */
} orc_tree;

static int cmp_pt(const void *a, const void *b) {
    const orc_pt *x = (const orc_pt *)a, *y = (const orc_pt *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

static int32_t new_node(orc_tree *T) {
    if (T->nnodes == T->cap) {
        T->cap = T->cap ? 2 * T->cap : 64;
        T->nodes = (orc_node *)realloc(T->nodes, sizeof(orc_node) * (size_t)T->cap);
    }
    memset(&T->nodes[T->nnodes], 0, sizeof(orc_node));
    return T->nnodes++;
}

/* splitUsingBit(P, b): first index in [lo, hi) whose key has bit b set;
 * a binary search because the range is Morton-sorted. */
static int64_t split_using_bit(const orc_tree *T, int64_t lo, int64_t hi, int b) {
    int64_t a = lo, z = hi;
    while (a < z) {
        int64_t mid = a + (z - a) / 2;
        if ((T->pts[mid].key >> b) & 1u) z = mid; else a = mid + 1;
    }
    return a;
}

static int msb64(uint64_t x) { int b = 63; while (!((x >> b) & 1u)) --b; return b; }

/* buildTree(P, b) (Alg. 1) with empty cuts skipped. */
static int32_t build_rec(orc_tree *T, int64_t lo, int64_t hi, int32_t parent) {
    int32_t v = new_node(T);
    orc_node *nd = &T->nodes[v];
    nd->lo = lo; nd->hi = hi; nd->parent = parent; nd->left = nd->right = -1;
    int dim = T->dim;
    if (hi - lo <= T->leaf_max || T->pts[lo].key == T->pts[hi - 1].key) {
        /* createLeaf(P): leaf rule = reading 1/2 */
        T->nodes[v].split = -1;
        for (int a = 0; a < dim; ++a) { T->nodes[v].bmin[a] = INT32_MAX; T->nodes[v].bmax[a] = INT32_MIN; }
        for (int64_t i = lo; i < hi; ++i) {
            T->leaf_of[i] = v;
            for (int a = 0; a < dim; ++a) {
                if (T->pts[i].c[a] < T->nodes[v].bmin[a]) T->nodes[v].bmin[a] = T->pts[i].c[a];
                if (T->pts[i].c[a] > T->nodes[v].bmax[a]) T->nodes[v].bmax[a] = T->pts[i].c[a];
            }
        }
        if (hi == lo) for (int a = 0; a < dim; ++a) { T->nodes[v].bmin[a] = 0; T->nodes[v].bmax[a] = -1; }
        return v;
    }
    /* highest differing bit = the first non-empty cut below the common prefix (reading 3) */
    int b = msb64(T->pts[lo].key ^ T->pts[hi - 1].key);
    int64_t s = split_using_bit(T, lo, hi, b);
    T->nodes[v].split = b;
    int32_t L = build_rec(T, lo, s, v);
    int32_t R = build_rec(T, s, hi, v);
    nd = &T->nodes[v];
    nd->left = L; nd->right = R;
    for (int a = 0; a < dim; ++a) {
        nd->bmin[a] = T->nodes[L].bmin[a] < T->nodes[R].bmin[a] ? T->nodes[L].bmin[a] : T->nodes[R].bmin[a];
        nd->bmax[a] = T->nodes[L].bmax[a] > T->nodes[R].bmax[a] ? T->nodes[L].bmax[a] : T->nodes[R].bmax[a];
    }
    return v;
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* Build from points (row-major int32 [n][dim]) with the given ids (NULL -> 0..n-1),
 * keys of `bits` bits per axis.  The random shift (§2, "select a random shift
 * ... kept throughout") is applied by the caller to the coordinates it passes, which
 * then need one more bit per axis (2D: 31). */
/* Keys of the levels bits-1 .. lo of every coordinate ((bits - lo) * dim key bits).
 * The 3D random shift (DESIGN reading R31) makes coordinates 22-bit; its key takes the
 * levels 21 .. 1 (63 bits: the Morton order of the shifted grid at cell size 2), with
 * the exact coordinates kept for every distance. */
orc_tree *orc_build_levels(const int32_t *pts, const int32_t *ids, int64_t n, int dim, int leaf_max, int bits,
                           int lo) {
    if ((dim != 2 && dim != 3) || n < 0 || leaf_max < 1 || bits < 1 || lo < 0 || lo >= bits ||
        (bits - lo) * dim > 64) return NULL;
    orc_tree *T = (orc_tree *)calloc(1, sizeof(orc_tree));
    T->dim = dim; T->leaf_max = leaf_max; T->n = n; T->bits = bits; T->lo = lo;
    T->pts = (orc_pt *)malloc(sizeof(orc_pt) * (size_t)(n ? n : 1));
    T->leaf_of = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    T->row_of = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        orc_pt *p = &T->pts[i];
        p->id = ids ? ids[i] : (int32_t)i;
        p->c[0] = pts[i * dim]; p->c[1] = pts[i * dim + 1]; p->c[2] = dim == 3 ? pts[i * dim + 2] : 0;
        p->key = key_levels(&pts[i * dim], dim, bits, lo);
    }
    qsort(T->pts, (size_t)n, sizeof(orc_pt), cmp_pt);
    T->root = build_rec(T, 0, n, -1);
    /* output row of each point = rank of its id among all ids (reading 21) */
    int32_t *sid = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) sid[i] = T->pts[i].id;
    qsort(sid, (size_t)n, sizeof(int32_t), cmp_i32);
    for (int64_t i = 0; i < n; ++i) {
        int32_t *f = (int32_t *)bsearch(&T->pts[i].id, sid, (size_t)n, sizeof(int32_t), cmp_i32);
        T->row_of[i] = f - sid;
    }
    free(sid);
    return T;
}

orc_tree *orc_build_bits(const int32_t *pts, const int32_t *ids, int64_t n, int dim, int leaf_max, int bits) {
    return orc_build_levels(pts, ids, n, dim, leaf_max, bits, 0);
}

orc_tree *orc_build(const int32_t *pts, const int32_t *ids, int64_t n, int dim, int leaf_max) {
    return orc_build_bits(pts, ids, n, dim, leaf_max, bits_per_axis(dim));
}

void orc_free(orc_tree *T) {
    if (!T) return;
    free(T->pts); free(T->nodes); free(T->leaf_of); free(T->row_of); free(T);
}

int64_t orc_size(const orc_tree *T) { return T->n; }
int32_t orc_num_nodes(const orc_tree *T) { return T->nnodes; }
int32_t orc_root(const orc_tree *T) { return T->root; }

/* Sorted keys, ids and coordinates (x, y, z-or-0). */
void orc_export_points(const orc_tree *T, uint64_t *keys, int32_t *ids, int32_t *coords3) {
    for (int64_t i = 0; i < T->n; ++i) {
        if (keys) keys[i] = T->pts[i].key;
        if (ids) ids[i] = T->pts[i].id;
        if (coords3) for (int a = 0; a < 3; ++a) coords3[i * 3 + a] = T->pts[i].c[a];
    }
}

/* Nodes in creation (DFS pre-)order: lo, hi, split (-1 = leaf), parent/left/right
 * (node indices, -1 = none) and bbox (bmin[0..2], bmax[0..2]). */
void orc_export_nodes(const orc_tree *T, int64_t *lohi, int32_t *split, int32_t *links, int32_t *bbox6) {
    for (int32_t v = 0; v < T->nnodes; ++v) {
        const orc_node *nd = &T->nodes[v];
        lohi[2 * v] = nd->lo; lohi[2 * v + 1] = nd->hi;
        split[v] = nd->split;
        links[3 * v] = nd->parent; links[3 * v + 1] = nd->left; links[3 * v + 2] = nd->right;
        for (int a = 0; a < 3; ++a) { bbox6[6 * v + a] = nd->bmin[a]; bbox6[6 * v + 3 + a] = nd->bmax[a]; }
    }
}

/* ---------------------------------------------------------------- query */

/* Work counters: leaf points scanned (own point included),
 * nodes entered by searchDown, ascents of searchUp, insertions into the k-best set
 * (fills and evictions), and evictions alone (insertions into a full set). */
enum { CNT_DIST = 0, CNT_BOX = 1, CNT_ASCENT = 2, CNT_REPL = 3, CNT_EVICT = 4, NCNT = 5 };

typedef struct {
    const orc_tree *T;
    const int32_t *q;   /* query coordinates */
    int32_t qid;        /* excluded id (reading 13); INT32_MIN = none */
    nset *N;
    int64_t cnt[NCNT];
} qctx;

static void scan_leaf(qctx *Q, const orc_node *nd) {
    for (int64_t i = nd->lo; i < nd->hi; ++i) {
        const orc_pt *p = &Q->T->pts[i];
        Q->cnt[CNT_DIST]++;
        if (p->id == Q->qid) continue;            /* "q != p" by id */
        int64_t d = dist2(Q->q, p->c, Q->T->dim);
        const int full = Q->N->cnt == Q->N->k;
        const int ins = nset_insert(Q->N, d, p->id);
        Q->cnt[CNT_REPL] += ins;
        Q->cnt[CNT_EVICT] += ins && full;
    }
}

/* searchDown(T, p, N) (Alg. 2). */
static void search_down(qctx *Q, int32_t v) {
    const orc_node *nd = &Q->T->nodes[v];
    Q->cnt[CNT_BOX]++;
    /* withinBox(T, p, r): prune iff |N| = k and boxd2 > r^2 (strict; reading 8) */
    if (orc_boxd2(Q->q, nd->bmin, nd->bmax, Q->T->dim) > nset_radius(Q->N)) return;
    if (nd->split < 0) { scan_leaf(Q, nd); return; }
    /* nearer child first (reading 10: by box distance, tie -> left) */
    const orc_node *L = &Q->T->nodes[nd->left], *R = &Q->T->nodes[nd->right];
    int64_t dl = orc_boxd2(Q->q, L->bmin, L->bmax, Q->T->dim);
    int64_t dr = orc_boxd2(Q->q, R->bmin, R->bmax, Q->T->dim);
    if (dl <= dr) { search_down(Q, nd->left); search_down(Q, nd->right); }
    else { search_down(Q, nd->right); search_down(Q, nd->left); }
}

/* not withinBox(C, p, -r) of Alg. 3, reading 9: with the tight bbox
 * [lo, hi] of C and q inside it, every point outside subtree(C) has d^2 >= m^2
 * where m = min margin + 1; stop iff m^2 > r^2.  q outside the box: never stop. */
static int stop_here(qctx *Q, const orc_node *C) {
    if (Q->N->cnt < Q->N->k) return 0;
    int64_t m = orc_margin(Q->q, C->bmin, C->bmax, Q->T->dim);
    if (m < 0) return 0;
    m += 1;
    return m * m > nset_radius(Q->N);
}

/* searchUp(C, p) (Alg. 3) from leaf c. */
static void search_up(qctx *Q, int32_t c) {
    const orc_tree *T = Q->T;
    scan_leaf(Q, &T->nodes[c]);
    while (T->nodes[c].parent >= 0) {
        if (stop_here(Q, &T->nodes[c])) break;
        int32_t P = T->nodes[c].parent;
        int32_t S = T->nodes[P].left == c ? T->nodes[P].right : T->nodes[P].left;
        search_down(Q, S);
        c = P;
        Q->cnt[CNT_ASCENT]++;
    }
}

/* Bit-based leaf location: descend by the query key's split bits. */
static int32_t locate_leaf(const orc_tree *T, uint64_t key) {
    int32_t v = T->root;
    while (T->nodes[v].split >= 0)
        v = ((key >> T->nodes[v].split) & 1u) ? T->nodes[v].right : T->nodes[v].left;
    return v;
}

static void write_row(const nset *N, int k, int32_t *oi, int64_t *od) {
    for (int j = 0; j < k; ++j) {
        if (j < N->cnt) { oi[j] = N->id[j]; od[j] = N->d[j]; }
        else { oi[j] = -1; od[j] = INT64_MAX; }   /* reading 15 */
    }
}

enum { MODE_LEAF = 0, MODE_ROOT = 1, MODE_EXT_BIT = 2, MODE_EXT_ROOT = 3 };

typedef struct {
    const orc_tree *T;
    int k, mode;
    int64_t begin, end;
    const int32_t *queries;  /* external queries (modes 2, 3) */
    int32_t *oi;
    int64_t *od;
    int64_t cnt[NCNT];
} job;

static void *run_job(void *arg) {
    job *J = (job *)arg;
    const orc_tree *T = J->T;
    int k = J->k;
    int64_t *dd = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    int32_t *ii = (int32_t *)malloc(sizeof(int32_t) * (size_t)k);
    memset(J->cnt, 0, sizeof(J->cnt));
    for (int64_t t = J->begin; t < J->end; ++t) {
        nset N = {k, 0, dd, ii};
        qctx Q;
        memset(&Q, 0, sizeof(Q));
        Q.T = T; Q.N = &N;
        int64_t row;
        int32_t qc[3] = {0, 0, 0};
        if (J->mode == MODE_LEAF || J->mode == MODE_ROOT) {
            const orc_pt *p = &T->pts[t];      /* queries in Morton order */
            Q.q = p->c; Q.qid = p->id;
            row = T->row_of[t];
            if (J->mode == MODE_LEAF) search_up(&Q, T->leaf_of[t]);
            else search_down(&Q, T->root);
        } else {
            for (int a = 0; a < T->dim; ++a) qc[a] = J->queries[t * T->dim + a];
            Q.q = qc; Q.qid = INT32_MIN;        /* dynamic query: nothing excluded */
            row = t;
            if (T->n == 0) { /* empty tree: nothing to search */ }
            else if (J->mode == MODE_EXT_BIT) search_up(&Q, locate_leaf(T, key_levels(qc, T->dim, T->bits, T->lo)));
            else search_down(&Q, T->root);
        }
        write_row(&N, k, J->oi + row * k, J->od + row * k);
        for (int c = 0; c < NCNT; ++c) J->cnt[c] += Q.cnt[c];
    }
    free(dd); free(ii);
    return NULL;
}

int orc_num_cores(void) {
    cpu_set_t s;
    if (sched_getaffinity(0, sizeof(s), &s) == 0) return CPU_COUNT(&s);
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

/* Contiguous chunks of the Morton-ordered query sequence per thread. */
static int run_parallel(const orc_tree *T, int k, int mode, int64_t m, const int32_t *queries,
                        int nthreads, int32_t *oi, int64_t *od, int64_t *counters) {
    if (k < 1) return -1;
    if (nthreads <= 0) nthreads = orc_num_cores();
    if (nthreads > m) nthreads = m > 0 ? (int)m : 1;
    job *jobs = (job *)calloc((size_t)nthreads, sizeof(job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (job){T, k, mode, m * t / nthreads, m * (t + 1) / nthreads, queries, oi, od, {0}};
        if (nthreads == 1) run_job(&jobs[t]); else pthread_create(&th[t], NULL, run_job, &jobs[t]);
    }
    if (nthreads > 1) for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    if (counters) {
        for (int c = 0; c < NCNT; ++c) counters[c] = 0;
        for (int t = 0; t < nthreads; ++t) for (int c = 0; c < NCNT; ++c) counters[c] += jobs[t].cnt[c];
    }
    free(jobs); free(th);
    return 0;
}

/* All-points k-NN graph, leaf-based.  Row r = r-th smallest live id. */
int orc_knn_all(const orc_tree *T, int k, int nthreads, int32_t *oi, int64_t *od, int64_t *counters) {
    return run_parallel(T, k, MODE_LEAF, T->n, NULL, nthreads, oi, od, counters);
}

/* Same, root-based (Alg. 2 from the root). */
int orc_knn_all_root(const orc_tree *T, int k, int nthreads, int32_t *oi, int64_t *od, int64_t *counters) {
    return run_parallel(T, k, MODE_ROOT, T->n, NULL, nthreads, oi, od, counters);
}

/* External ("dynamic") queries: bit-based (root_based = 0) or
 * root-based (1).  Row j = query j.  No self-exclusion. */
int orc_knn_queries(const orc_tree *T, const int32_t *queries, int64_t m, int k, int root_based,
                    int nthreads, int32_t *oi, int64_t *od, int64_t *counters) {
    return run_parallel(T, k, root_based ? MODE_EXT_ROOT : MODE_EXT_BIT, m, queries, nthreads, oi, od, counters);
}

/* --------------------------------------------------------- brute force */

typedef struct {
    const int32_t *pts, *ids;
    int64_t n;
    int dim, k;
    const int32_t *qpts;       /* query coordinates [nq][dim] */
    const int32_t *qids;       /* excluded id per query, or NULL */
    int64_t begin, end;
    int32_t *oi;
    int64_t *od;
} bjob;

static void *run_brute(void *arg) {
    bjob *J = (bjob *)arg;
    int64_t *dd = (int64_t *)malloc(sizeof(int64_t) * (size_t)J->k);
    int32_t *ii = (int32_t *)malloc(sizeof(int32_t) * (size_t)J->k);
    for (int64_t t = J->begin; t < J->end; ++t) {
        nset N = {J->k, 0, dd, ii};
        const int32_t *q = J->qpts + t * J->dim;
        int32_t qid = J->qids ? J->qids[t] : INT32_MIN;
        for (int64_t j = 0; j < J->n; ++j) {
            int32_t id = J->ids ? J->ids[j] : (int32_t)j;
            if (id == qid) continue;
            nset_insert(&N, dist2(q, J->pts + j * J->dim, J->dim), id);
        }
        write_row(&N, J->k, J->oi + t * J->k, J->od + t * J->k);
    }
    free(dd); free(ii);
    return NULL;
}

/* The plain definition (SURVEY §8(c) "Result definition"): for each query t,
 * the first min(k, |others|) elements of {(d^2(q_t, p_j), id_j) : id_j != qid_t}
 * in lexicographic order, padded with (-1, INT64_MAX). */
int orc_brute_knn(const int32_t *pts, const int32_t *ids, int64_t n, int dim,
                  const int32_t *qpts, const int32_t *qids, int64_t nq, int k,
                  int nthreads, int32_t *oi, int64_t *od) {
    if (k < 1) return -1;
    if (nthreads <= 0) nthreads = orc_num_cores();
    if (nthreads > nq) nthreads = nq > 0 ? (int)nq : 1;
    bjob *jobs = (bjob *)calloc((size_t)nthreads, sizeof(bjob));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (bjob){pts, ids, n, dim, k, qpts, qids, nq * t / nthreads, nq * (t + 1) / nthreads, oi, od};
        if (nthreads == 1) run_brute(&jobs[t]); else pthread_create(&th[t], NULL, run_brute, &jobs[t]);
    }
    if (nthreads > 1) for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs); free(th);
    return 0;
}
