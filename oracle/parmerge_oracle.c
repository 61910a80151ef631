/*
 * parmerge_oracle.c -- CPU restatement of the reference's merge path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
 * leg (cpu_baseline / --impl reference) load it, and only as the checker or
 * as the timed CPU baseline.
 *
 * Each function restates one routine of the reference package
 * `parmerge` (/root/reference/pkg/src/parmerge) in plain C and cites the
 * file:line it follows.  Keys are signed integers of 4 or 8 bytes (the
 * reference's KeyedArray is int32 only, records.py:9; its numba kernels are
 * type generic and are called with int64 arrays for the skewed config, see
 * SURVEY.md 0.5).  The payload is an opaque row of `w` bytes per record that
 * travels with its key (records.py:15-22).
 *
 * Pinned by tests/test_oracle.py against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py) and against the known-answer
 * examples in the reference's own tests.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define SCRATCH_RECORDS 256 /* _kernels.py:17 */
#define SCRATCH_MAX_WIDTH 60 /* _kernels.py:18 */

static inline void swap_rows(uint8_t *p, int64_t w, int64_t i, int64_t j) {
    uint8_t *a = p + i * w, *b = p + j * w;
    for (int64_t c = 0; c < w; ++c) { uint8_t t = a[c]; a[c] = b[c]; b[c] = t; }
}

#define DEFINE_ORACLE(KT, SUF)                                                   \
/* _kernels.py:22-30 */                                                          \
int64_t orc_lower_bound_##SUF(const KT *k, int64_t lo, int64_t hi, KT v) {       \
    while (lo < hi) { int64_t mid = (lo + hi) >> 1;                              \
        if (k[mid] < v) lo = mid + 1; else hi = mid; }                           \
    return lo; }                                                                 \
/* _kernels.py:34-42 */                                                          \
int64_t orc_upper_bound_##SUF(const KT *k, int64_t lo, int64_t hi, KT v) {       \
    while (lo < hi) { int64_t mid = (lo + hi) >> 1;                              \
        if (k[mid] <= v) lo = mid + 1; else hi = mid; }                          \
    return lo; }                                                                 \
/* median.py:23-60 (Alg. 1, double binary search; equal pivots stop early) */    \
void orc_find_median_##SUF(const KT *a, int64_t la, const KT *b, int64_t lb,     \
                           int64_t *out) {                                       \
    if (la == 0 || lb == 0 || a[la - 1] <= b[0]) { out[0] = la; out[1] = 0; return; } \
    if (!(a[0] <= b[lb - 1])) { out[0] = 0; out[1] = lb; return; }               \
    int64_t left_a = 0, limit_a = la, left_b = 0, limit_b = lb, pa, pb;          \
    while (left_a < limit_a && left_b < limit_b) {                               \
        pa = (limit_a - left_a) / 2 + left_a;                                    \
        pb = (limit_b - left_b) / 2 + left_b;                                    \
        KT va = a[pa], vb = b[pb];                                               \
        if (va == vb) break;                                                     \
        if (va < vb) {                                                           \
            if (pa + pb < (la - pa) + (lb - pb)) left_a = pa + 1;                \
            else limit_b = pb;                                                   \
        } else {                                                                 \
            if (pa + pb < (la - pa) + (lb - pb)) left_b = pb + 1;                \
            else limit_a = pa;                                                   \
        }                                                                        \
    }                                                                            \
    out[0] = (limit_a - left_a) / 2 + left_a;                                    \
    out[1] = (limit_b - left_b) / 2 + left_b; }                                  \
/* _kernels.py:46-88 */                                                          \
static void staged_exchange_##SUF(KT *k, uint8_t *p, int64_t w, int64_t lo,      \
                                  int64_t la, int64_t lb) {                      \
    KT sk[SCRATCH_RECORDS]; uint8_t sp[SCRATCH_RECORDS * SCRATCH_MAX_WIDTH];     \
    if (la <= lb) {                                                              \
        memcpy(sk, k + lo, la * sizeof(KT)); memcpy(sp, p + lo * w, la * w);     \
        memmove(k + lo, k + lo + la, lb * sizeof(KT));                           \
        memmove(p + lo * w, p + (lo + la) * w, lb * w);                          \
        memcpy(k + lo + lb, sk, la * sizeof(KT)); memcpy(p + (lo + lb) * w, sp, la * w); \
    } else {                                                                     \
        memcpy(sk, k + lo + la, lb * sizeof(KT)); memcpy(sp, p + (lo + la) * w, lb * w); \
        memmove(k + lo + lb, k + lo, la * sizeof(KT));                           \
        memmove(p + (lo + lb) * w, p + lo * w, la * w);                          \
        memcpy(k + lo, sk, lb * sizeof(KT)); memcpy(p + lo * w, sp, lb * w);     \
    } }                                                                          \
/* _kernels.py:92-150 (linear shifting: staged path, else Gries-Mills sweeps) */ \
void orc_linear_shift_##SUF(KT *k, uint8_t *p, int64_t w, int64_t lo,            \
                            int64_t len_a, int64_t len_b) {                      \
    int64_t la = len_a, lb = len_b, hi = lo + la + lb;                           \
    while (la > 0 && lb > 0) {                                                   \
        if ((la < lb ? la : lb) <= SCRATCH_RECORDS && w <= SCRATCH_MAX_WIDTH) {  \
            staged_exchange_##SUF(k, p, w, lo, la, lb); return; }                \
        if (la <= lb) {                                                          \
            int64_t base = hi - la;                                              \
            for (int64_t i = 0; i < la; ++i) {                                   \
                KT t = k[lo + i]; k[lo + i] = k[base + i]; k[base + i] = t;      \
                if (w) swap_rows(p, w, lo + i, base + i); }                      \
            hi -= la; lb -= la;                                                  \
        } else {                                                                 \
            int64_t base = lo + la;                                              \
            for (int64_t i = lb - 1; i >= 0; --i) {                              \
                KT t = k[lo + i]; k[lo + i] = k[base + i]; k[base + i] = t;      \
                if (w) swap_rows(p, w, lo + i, base + i); }                      \
            lo += lb; la -= lb;                                                  \
        }                                                                        \
    } }                                                                          \
/* _kernels.py:154-197 (circular shifting: gcd cycles, one spare record) */      \
void orc_circular_shift_##SUF(KT *k, uint8_t *p, int64_t w, int64_t lo,          \
                              int64_t len_a, int64_t len_b) {                    \
    if (len_a == 0 || len_b == 0) return;                                        \
    int64_t g = len_a, h = len_b;                                                \
    while (h) { int64_t t = g % h; g = h; h = t; }                               \
    uint8_t *tp = (uint8_t *)malloc(w ? w : 1), *sb = (uint8_t *)malloc(w ? w : 1); \
    for (int64_t c = 0; c < g; ++c) {                                            \
        KT tk = k[lo + c]; if (w) memcpy(tp, p + (lo + c) * w, w);               \
        int64_t j = c < len_a ? c + len_b : c - len_a;                           \
        while (j != c) {                                                         \
            int64_t q = lo + j; KT s = k[q]; k[q] = tk; tk = s;                  \
            if (w) { memcpy(sb, p + q * w, w); memcpy(p + q * w, tp, w); memcpy(tp, sb, w); } \
            j = j < len_a ? j + len_b : j - len_a;                               \
        }                                                                        \
        k[lo + c] = tk; if (w) memcpy(p + (lo + c) * w, tp, w);                  \
    }                                                                            \
    free(tp); free(sb); }                                                        \
/* _kernels.py:201-223 (O(1)-space stable rotation merge) */                     \
void orc_rotation_merge_##SUF(KT *k, uint8_t *p, int64_t w, int64_t start,       \
                              int64_t middle, int64_t end, int circular) {       \
    int64_t s = start, m = middle, e = end;                                      \
    while (s < m && m < e) {                                                     \
        s = orc_upper_bound_##SUF(k, s, m, k[m]);                                \
        if (s == m) break;                                                       \
        int64_t k_end = orc_lower_bound_##SUF(k, m, e, k[s]);                    \
        if (circular) orc_circular_shift_##SUF(k, p, w, s, m - s, k_end - m);    \
        else orc_linear_shift_##SUF(k, p, w, s, m - s, k_end - m);               \
        s += k_end - m; m = k_end;                                               \
    } }                                                                          \
/* _kernels.py:227-313 (stable buffered merge, min-side scratch; A wins ties) */ \
void orc_buffered_merge_##SUF(KT *k, uint8_t *p, int64_t w, int64_t start,       \
                              int64_t middle, int64_t end, KT *bk, uint8_t *bp) {\
    int64_t la = middle - start, lb = end - middle;                              \
    if (la == 0 || lb == 0) return;                                              \
    if (la <= lb) {                                                              \
        memcpy(bk, k + start, la * sizeof(KT)); memcpy(bp, p + start * w, la * w); \
        int64_t i = 0, j = middle, d = start;                                    \
        while (i < la && j < end) {                                              \
            if (k[j] < bk[i]) { k[d] = k[j]; if (w) memcpy(p + d * w, p + j * w, w); ++j; } \
            else { k[d] = bk[i]; if (w) memcpy(p + d * w, bp + i * w, w); ++i; } \
            ++d; }                                                               \
        while (i < la) { k[d] = bk[i]; if (w) memcpy(p + d * w, bp + i * w, w); ++i; ++d; } \
    } else {                                                                     \
        memcpy(bk, k + middle, lb * sizeof(KT)); memcpy(bp, p + middle * w, lb * w); \
        int64_t i = lb - 1, j = middle - 1, d = end - 1;                         \
        while (i >= 0 && j >= start) {                                           \
            if (bk[i] >= k[j]) { k[d] = bk[i]; if (w) memcpy(p + d * w, bp + i * w, w); --i; } \
            else { k[d] = k[j]; if (w) memcpy(p + d * w, p + j * w, w); --j; }   \
            --d; }                                                               \
        while (i >= 0) { k[d] = bk[i]; if (w) memcpy(p + d * w, bp + i * w, w); --i; --d; } \
    } }                                                                          \
/* seqmerge.py:55-75: allocate the min-side scratch and merge */                 \
int orc_seq_merge_buffered_##SUF(KT *k, uint8_t *p, int64_t w, int64_t start,    \
                                 int64_t middle, int64_t end) {                  \
    int64_t need = middle - start < end - middle ? middle - start : end - middle;\
    KT *bk = (KT *)malloc((need ? need : 1) * sizeof(KT));                       \
    uint8_t *bp = (uint8_t *)malloc((need != 0 && w != 0) ? (size_t)(need * w) : 1);                    \
    if (!bk || !bp) { free(bk); free(bp); return -1; }                           \
    orc_buffered_merge_##SUF(k, p, w, start, middle, end, bk, bp);               \
    free(bk); free(bp); return 0; }                                              \
/* stable merge-path split on diagonal d of runs a[0,la), b[0,lb):              \
 * number of a-records among the first d outputs of the stable (a-first) merge */ \
int64_t orc_merge_path_##SUF(const KT *a, int64_t la, const KT *b, int64_t lb,   \
                             int64_t d) {                                        \
    int64_t lo = d > lb ? d - lb : 0, hi = d < la ? d : la;                      \
    while (lo < hi) { int64_t mid = (lo + hi) >> 1;                              \
        /* a[mid] is among the first d iff a[mid] <= b[d-1-mid] */               \
        if (a[mid] <= b[d - 1 - mid]) lo = mid + 1; else hi = mid; }             \
    return lo; }

DEFINE_ORACLE(int32_t, i32)
DEFINE_ORACLE(int64_t, i64)

/* ----------------------------------------------------------------------------
 * CPU baseline: merge_srecpar with a buffered leaf core on host threads.
 * srecpar.py:33-84 -- split with find_median, exchange the center blocks with
 * linear shifting, hand the right pair to another worker, recurse left, merge
 * the leaves with seq_merge_buffered (the "fastest reference CPU path",
 * SURVEY.md 6).  Threads stand in for the reference's ThreadPoolExecutor
 * (_pool.py:14-31); every task owns a disjoint interval.
 * -------------------------------------------------------------------------- */
typedef struct {
    void *k; uint8_t *p; int64_t w; int64_t s, m, e; int level, depth;
    int64_t size_limit; int key_bytes;
    int leaf;  /* 0: seq_merge_buffered leaves; 1: the default rotation leaves (seqmerge.py:37-52) */
} rp_task;

static void *rp_core(void *arg);

static void rp_run(rp_task *t) {
    pthread_t tids[64]; rp_task subs[64]; int ns = 0;
    int64_t start = t->s, middle = t->m, end = t->e; int level = t->level;
    if (start == middle || middle == end) return;
    while (level != t->depth && (end - start) > t->size_limit) {
        int64_t piv[2];
        if (t->key_bytes == 4) {
            int32_t *k = (int32_t *)t->k;
            orc_find_median_i32(k + start, middle - start, k + middle, end - middle, piv);
        } else {
            int64_t *k = (int64_t *)t->k;
            orc_find_median_i64(k + start, middle - start, k + middle, end - middle, piv);
        }
        int64_t rest_a = (middle - start) - piv[0];
        if (t->key_bytes == 4)
            orc_linear_shift_i32((int32_t *)t->k, t->p, t->w, start + piv[0], rest_a, piv[1]);
        else
            orc_linear_shift_i64((int64_t *)t->k, t->p, t->w, start + piv[0], rest_a, piv[1]);
        int64_t rs = start + piv[0] + piv[1];
        subs[ns] = *t; subs[ns].s = rs; subs[ns].m = rs + rest_a; subs[ns].e = end;
        subs[ns].level = level + 1;
        if (pthread_create(&tids[ns], NULL, rp_core, &subs[ns]) != 0) {
            rp_run(&subs[ns]); tids[ns] = 0; }
        ++ns;
        end = rs; middle = start + piv[0]; ++level;
    }
    if (t->leaf == 1) {  /* seq_merge_rotation(arr, job, LINEAR), srecpar.py:57 default leaf */
        if (t->key_bytes == 4)
            orc_rotation_merge_i32((int32_t *)t->k, t->p, t->w, start, middle, end, 0);
        else
            orc_rotation_merge_i64((int64_t *)t->k, t->p, t->w, start, middle, end, 0);
    } else if (t->key_bytes == 4)
        orc_seq_merge_buffered_i32((int32_t *)t->k, t->p, t->w, start, middle, end);
    else
        orc_seq_merge_buffered_i64((int64_t *)t->k, t->p, t->w, start, middle, end);
    for (int i = 0; i < ns; ++i) if (tids[i]) pthread_join(tids[i], NULL);
}

static void *rp_core(void *arg) { rp_run((rp_task *)arg); return NULL; }

/* merge_srecpar(arr, job, threads, leaf_core=...), srecpar.py:33-60; leaf 0 =
 * seq_merge_buffered (the fastest reference path), 1 = the default rotation leaves */
int orc_srecpar(void *keys, int key_bytes, uint8_t *payload, int64_t w,
                int64_t start, int64_t middle, int64_t end, int threads,
                int64_t size_limit, int leaf) {
    if (threads < 1 || (threads & (threads - 1))) return -1;
    if (start == middle || middle == end) return 0;
    if (key_bytes == 4) { int32_t *k = (int32_t *)keys; if (k[middle - 1] <= k[middle]) return 0; }
    else { int64_t *k = (int64_t *)keys; if (k[middle - 1] <= k[middle]) return 0; }
    int depth = 0; while ((1 << (depth + 1)) <= threads) ++depth;
    rp_task t = {keys, payload, w, start, middle, end, 0, depth, size_limit, key_bytes, leaf};
    rp_run(&t);
    return 0;
}

int orc_srecpar_buffered(void *keys, int key_bytes, uint8_t *payload, int64_t w,
                         int64_t start, int64_t middle, int64_t end, int threads,
                         int64_t size_limit) {
    return orc_srecpar(keys, key_bytes, payload, w, start, middle, end, threads, size_limit, 0);
}
