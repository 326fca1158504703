/*
 * saix_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference `saix` package's hot path
 * (DC3 suffix array, Kasai LCP, sparse-table RMQ, lcp_query and the
 * generalized-suffix-array longest-overlap scan).  It exists to check the
 * CUDA implementation and to time the reference algorithm on the host
 * (`bench.py` cpu_baseline / --impl reference, kind "port").  Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU legs may load it; the product
 * path (paper_1404_3448_b200) never links or calls this file.
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to the reference checkout (pkg/src/saix/...).  The restatement
 * is pinned against the reference's own golden vectors and against outputs
 * of the reference itself (tests/golden/, made by tests/golden/make_golden.py).
 */
#include <malloc.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ */
/* small helpers                                                        */
/* ------------------------------------------------------------------ */

/* Keep freed buffers on the heap instead of returning them to the kernel
 * (the reference does the same for timing, bench.py:59-72 tune_allocator):
 * otherwise every per-pair DC3 mmaps/munmaps its arrays and host threads
 * serialise on the kernel's mm lock. */
__attribute__((constructor)) static void tune_allocator(void) {
    mallopt(M_MMAP_THRESHOLD, 1 << 30);
    mallopt(M_TRIM_THRESHOLD, 1 << 30);
}

static void *xcalloc(size_t n, size_t sz) {
    void *p = calloc(n ? n : 1, sz);
    if (!p) abort();
    return p;
}

/* Stable counting pass: reorder `order` by keys[order] (suffix_index.py:156-170). */
static void counting_reorder(const int32_t *keys, int32_t *order, int64_t len,
                             int64_t key_bound, int32_t *scratch) {
    int64_t *counts = xcalloc((size_t)key_bound + 2, sizeof(int64_t));
    for (int64_t i = 0; i < len; i++) counts[keys[order[i]] + 1]++;
    for (int64_t v = 1; v < key_bound + 2; v++) counts[v] += counts[v - 1];
    for (int64_t i = 0; i < len; i++) {
        int32_t k = keys[order[i]];
        scratch[counts[k]++] = order[i];
    }
    memcpy(order, scratch, (size_t)len * sizeof(int32_t));
    free(counts);
}

/* ------------------------------------------------------------------ */
/* DC3 (suffix_index.py:143-392)                                        */
/* ------------------------------------------------------------------ */

typedef struct {
    /* level-0 introspection, Dc3Workspace (suffix_index.py:119-140) */
    int32_t *triple_text;       /* m entries                           */
    int32_t *sample_rank;       /* n+3 entries, 1-based, 0 elsewhere   */
    int32_t *sorted_samples;    /* real samples (< n) in rank order    */
    int64_t n_sorted_samples;
    int32_t *sorted_nonsamples; /* mod-0 positions in order            */
    int64_t n_sorted_nonsamples;
    int32_t depth;
} oracle_probe;

/* _sample_positions (suffix_index.py:149-153) */
static void sample_counts(int64_t n, int64_t *m1, int64_t *m2) {
    int64_t limit = (n % 3 == 1) ? n + 1 : n;
    *m1 = limit > 1 ? (limit - 1 + 2) / 3 : 0;
    *m2 = limit > 2 ? (limit - 2 + 2) / 3 : 0;
}

static int32_t *dc3_rec(const int32_t *t, int64_t n, int64_t sigma,
                        int32_t *depth_out, oracle_probe *probe);

/* _name_triples + _sort_samples (suffix_index.py:221-271).  Sorting is a
 * three-pass LSD counting sort over the (t[s], t[s+1], t[s+2]) components;
 * any exact sort yields the same dense names (equal triples get equal names
 * and recursion fixes their order, suffix_index.py:75-80). */
static int32_t *sort_samples(const int32_t *tp, int64_t n, int64_t sigma,
                             int32_t *rank_of, int32_t *depth,
                             int32_t **triple_text_out, int64_t *m_out) {
    int64_t m1, m2;
    sample_counts(n, &m1, &m2);
    int64_t m = m1 + m2;
    *m_out = m;
    *depth = 0;
    int32_t *s12 = xcalloc((size_t)m, sizeof(int32_t));
    for (int64_t j = 0; j < m1; j++) s12[j] = (int32_t)(3 * j + 1);
    for (int64_t j = 0; j < m2; j++) s12[m1 + j] = (int32_t)(3 * j + 2);
    int32_t *sorted12 = xcalloc((size_t)m, sizeof(int32_t));
    int32_t *scratch = xcalloc((size_t)m, sizeof(int32_t));
    memcpy(sorted12, s12, (size_t)m * sizeof(int32_t));
    /* least significant component first; keys are read through tp+offset */
    for (int c = 2; c >= 0; c--) counting_reorder(tp + c, sorted12, m, sigma, scratch);
    /* dense names in sorted order (suffix_index.py:239-252) */
    int32_t *name_of = xcalloc((size_t)n + 3, sizeof(int32_t));
    int32_t name = 0;
    for (int64_t r = 0; r < m; r++) {
        int32_t p = sorted12[r];
        if (r == 0) {
            name = 1;
        } else {
            int32_t q = sorted12[r - 1];
            if (tp[p] != tp[q] || tp[p + 1] != tp[q + 1] || tp[p + 2] != tp[q + 2]) name++;
        }
        name_of[p] = name;
    }
    int32_t distinct = name;
    int32_t *triple_text = xcalloc((size_t)m, sizeof(int32_t));
    for (int64_t s = 0; s < m; s++) triple_text[s] = name_of[s12[s]];
    free(name_of);
    if (distinct < m) {
        int32_t d = 0;
        int32_t *sa_rec = dc3_rec(triple_text, m, distinct, &d, NULL);
        *depth = d + 1;
        for (int64_t r = 0; r < m; r++) sorted12[r] = s12[sa_rec[r]];
        free(sa_rec);
    }
    for (int64_t r = 0; r < m; r++) rank_of[sorted12[r]] = (int32_t)(r + 1);
    free(s12);
    free(scratch);
    if (triple_text_out) *triple_text_out = triple_text; else free(triple_text);
    return sorted12;
}

/* _merge_walk (suffix_index.py:173-218) */
static void merge_walk(const int32_t *tp, const int32_t *rank_of,
                       const int32_t *a, int64_t m, const int32_t *b, int64_t k,
                       int32_t *out) {
    int64_t i = 0, j = 0, w = 0;
    while (i < m && j < k) {
        int32_t x = a[i], y = b[j];
        int a_first;
        if (tp[x] != tp[y]) a_first = tp[x] < tp[y];
        else if (x % 3 == 1) a_first = rank_of[x + 1] < rank_of[y + 1];
        else if (tp[x + 1] != tp[y + 1]) a_first = tp[x + 1] < tp[y + 1];
        else a_first = rank_of[x + 2] < rank_of[y + 2];
        out[w++] = a_first ? a[i++] : b[j++];
    }
    while (i < m) out[w++] = a[i++];
    while (j < k) out[w++] = b[j++];
}

/* _dc3 (suffix_index.py:381-392) */
static int32_t *dc3_rec(const int32_t *t, int64_t n, int64_t sigma,
                        int32_t *depth_out, oracle_probe *probe) {
    *depth_out = 0;
    if (n == 0) return xcalloc(1, sizeof(int32_t));
    if (n == 1) return xcalloc(1, sizeof(int32_t));
    int32_t *tp = xcalloc((size_t)n + 3, sizeof(int32_t)); /* _padded 143-146 */
    memcpy(tp, t, (size_t)n * sizeof(int32_t));
    int32_t *rank_of = xcalloc((size_t)n + 3, sizeof(int32_t));
    int64_t m;
    int32_t depth;
    int32_t *triple_text = NULL;
    int32_t *sorted12 = sort_samples(tp, n, sigma, rank_of, &depth,
                                     probe ? &triple_text : NULL, &m);
    /* _sort_nonsamples (274-290): mod-1 samples in rank order, minus one,
     * then a stable counting pass on the first character. */
    int64_t k = 0;
    int32_t *sorted0 = xcalloc((size_t)m + 1, sizeof(int32_t));
    for (int64_t r = 0; r < m; r++)
        if (sorted12[r] % 3 == 1) sorted0[k++] = sorted12[r] - 1;
    int32_t *scratch = xcalloc((size_t)k + 1, sizeof(int32_t));
    counting_reorder(tp, sorted0, k, sigma, scratch);
    free(scratch);
    /* drop the padding sample (391) */
    int64_t ms = 0;
    int32_t *real = xcalloc((size_t)m + 1, sizeof(int32_t));
    for (int64_t r = 0; r < m; r++)
        if (sorted12[r] < n) real[ms++] = sorted12[r];
    int32_t *out = xcalloc((size_t)n, sizeof(int32_t));
    merge_walk(tp, rank_of, real, ms, sorted0, k, out);
    if (probe) {
        memcpy(probe->triple_text, triple_text, (size_t)m * sizeof(int32_t));
        memcpy(probe->sample_rank, rank_of, (size_t)(n + 3) * sizeof(int32_t));
        memcpy(probe->sorted_samples, real, (size_t)ms * sizeof(int32_t));
        probe->n_sorted_samples = ms;
        memcpy(probe->sorted_nonsamples, sorted0, (size_t)k * sizeof(int32_t));
        probe->n_sorted_nonsamples = k;
        probe->depth = depth;
        free(triple_text);
    }
    *depth_out = depth;
    free(tp);
    free(rank_of);
    free(sorted12);
    free(sorted0);
    free(real);
    return out;
}

/* build_sa_dc3 + SuffixArray.from_order (suffix_index.py:395-399, 96-101).
 * sa/rank may be NULL.  probe arrays (when probe != NULL) must hold
 * m, n+3, m, ceil(n/3) entries. */
EXPORT int oracle_dc3(const int32_t *text, int64_t n, int64_t sigma,
                      int64_t *sa, int64_t *rank, oracle_probe *probe) {
    if (n < 0 || n >= (int64_t)1 << 31) return -1;
    int32_t depth;
    if (probe && n <= 1) {
        /* prepare_dc3_workspace on n <= 1 (suffix_index.py:434-449) */
        int64_t m1, m2;
        sample_counts(n, &m1, &m2);
        memset(probe->sample_rank, 0, (size_t)(n + 3) * sizeof(int32_t));
        probe->n_sorted_samples = 0;
        probe->n_sorted_nonsamples = n;
        probe->depth = 0;
        if (n == 1) {
            probe->triple_text[0] = 1;   /* the padding position 1 names (0,0,0) */
            probe->sample_rank[1] = 1;
            probe->sorted_nonsamples[0] = 0;
        }
    }
    int32_t *order = dc3_rec(text, n, sigma, &depth, n > 1 ? probe : NULL);
    for (int64_t i = 0; i < n; i++) {
        if (sa) sa[i] = order[i];
        if (rank) rank[order[i]] = i;
    }
    free(order);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Kasai LCP (suffix_index.py:460-506)                                  */
/* ------------------------------------------------------------------ */

EXPORT int oracle_lcp(const int32_t *t, int64_t n, const int64_t *sa,
                      const int64_t *rank, int64_t *lcp) {
    int64_t h = 0;
    for (int64_t i = 0; i < n; i++) lcp[i] = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t r = rank[i];
        if (r > 0) {
            int64_t j = sa[r - 1];
            while (i + h < n && j + h < n && t[i + h] == t[j + h]) h++;
            lcp[r] = h;
            if (h) h--;
        } else {
            h = 0;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Sparse table RMQ (rmq.py:24-58, 254-259)                             */
/* ------------------------------------------------------------------ */

/* Number of table levels the reference builds for n values (rmq.py:38-47). */
EXPORT int64_t oracle_sparse_levels(int64_t n) {
    if (n <= 0) return 0;
    int64_t levels = 0;
    while (((int64_t)1 << levels) <= n) levels++;  /* == n.bit_length() */
    return levels < 1 ? 1 : levels;
}

/* Table layout: level k (len n-2^k+1) at offset sum_{k'<k}(n-2^k'+1). */
EXPORT int oracle_sparse_build(const int64_t *v, int64_t n, int64_t *table) {
    if (n <= 0) return -1;
    int64_t levels = oracle_sparse_levels(n);
    for (int64_t i = 0; i < n; i++) table[i] = i;
    int64_t off_prev = 0, off = n;
    for (int64_t k = 1; k < levels; k++) {
        int64_t len = n - ((int64_t)1 << k) + 1;
        if (len <= 0) break;
        int64_t half = (int64_t)1 << (k - 1);
        for (int64_t i = 0; i < len; i++) {
            int64_t l = table[off_prev + i], r = table[off_prev + i + half];
            table[off + i] = v[l] <= v[r] ? l : r;
        }
        off_prev = off;
        off += len;
    }
    return 0;
}

static int64_t level_offset(int64_t n, int64_t k) {
    int64_t off = 0;
    for (int64_t q = 0; q < k; q++) off += n - ((int64_t)1 << q) + 1;
    return off;
}

/* SparseTable.query (rmq.py:52-58); returns -1 on any out-of-range pair
 * (the reference raises IndexError, rmq.py:24-27). */
EXPORT int oracle_sparse_query(const int64_t *v, int64_t n, const int64_t *table,
                               const int64_t *qi, const int64_t *qj, int64_t q,
                               int64_t *out) {
    int64_t offs[64];
    int64_t levels = oracle_sparse_levels(n);
    for (int64_t k = 0; k < levels; k++) offs[k] = level_offset(n, k);
    for (int64_t t = 0; t < q; t++) {
        int64_t i = qi[t], j = qj[t];
        if (i < 0 || i >= n || j < 0 || j >= n) return -1;
        if (i > j) { int64_t x = i; i = j; j = x; }
        int64_t span = j - i + 1, k = 0;
        while (((int64_t)2 << k) <= span) k++;
        int64_t a = table[offs[k] + i];
        int64_t b = table[offs[k] + j - ((int64_t)1 << k) + 1];
        out[t] = v[a] <= v[b] ? a : b;
    }
    return 0;
}

/* Leftmost argmin by definition (tests/oracles.py:35-43), computed with a
 * block decomposition so that large-n checks need O(n) memory.  Same answer
 * as the sparse table by definition; used only where a 27-level table would
 * not fit in host RAM. */
EXPORT int oracle_argmin_blocked(const int64_t *v, int64_t n, const int64_t *qi,
                                 const int64_t *qj, int64_t q, int64_t *out) {
    const int64_t B = 256;
    int64_t nb = (n + B - 1) / B;
    int64_t *bmin = xcalloc((size_t)nb, sizeof(int64_t));
    for (int64_t b = 0; b < nb; b++) {
        int64_t best = b * B;
        for (int64_t i = b * B + 1; i < n && i < (b + 1) * B; i++)
            if (v[i] < v[best]) best = i;
        bmin[b] = best;
    }
    for (int64_t t = 0; t < q; t++) {
        int64_t i = qi[t], j = qj[t];
        if (i < 0 || i >= n || j < 0 || j >= n) { free(bmin); return -1; }
        if (i > j) { int64_t x = i; i = j; j = x; }
        int64_t best = i, bi = i / B, bj = j / B;
        if (bi == bj) {
            for (int64_t x = i + 1; x <= j; x++) if (v[x] < v[best]) best = x;
        } else {
            for (int64_t x = i + 1; x < (bi + 1) * B; x++) if (v[x] < v[best]) best = x;
            for (int64_t b = bi + 1; b < bj; b++) if (v[bmin[b]] < v[best]) best = bmin[b];
            for (int64_t x = bj * B; x <= j; x++) if (v[x] < v[best]) best = x;
        }
        out[t] = best;
    }
    free(bmin);
    return 0;
}

/* Leftmost argmin over inclusive [i, j] (swapped if i > j) -- the answer of
 * SparseTable.query (rmq.py:52-58, ties to the left operand) -- for large
 * query sweeps: 64-element blocks, a sparse table over the block minima
 * (the same leftmost combine rule), in-block scans at both ends; `threads`
 * pthreads split the queries.  Returns -1 on an out-of-range query. */
typedef struct {
    const int64_t *v, *qi, *qj, *bmin, *tab;
    int64_t n, nb, lo, hi;
    int64_t *out;
    int bad;
} ArgminJob;

#define AB_SHIFT 6
static int64_t ab_pick(const int64_t *v, int64_t a, int64_t b) { return v[a] <= v[b] ? a : b; }

static void *argmin_worker(void *p) {
    ArgminJob *J = (ArgminJob *)p;
    const int64_t *v = J->v;
    for (int64_t t = J->lo; t < J->hi; t++) {
        int64_t i = J->qi[t], j = J->qj[t];
        if (i < 0 || i >= J->n || j < 0 || j >= J->n) { J->bad = 1; return NULL; }
        if (i > j) { int64_t x = i; i = j; j = x; }
        int64_t bi = i >> AB_SHIFT, bj = j >> AB_SHIFT, best = i;
        if (bi == bj) {
            for (int64_t x = i + 1; x <= j; x++) if (v[x] < v[best]) best = x;
        } else {
            int64_t end = (bi + 1) << AB_SHIFT;
            for (int64_t x = i + 1; x < end; x++) if (v[x] < v[best]) best = x;
            if (bi + 1 <= bj - 1) {
                int64_t l = bi + 1, r = bj - 1, len = r - l + 1, k = 63 - __builtin_clzll((uint64_t)len);
                int64_t m = ab_pick(v, J->tab[k * J->nb + l], J->tab[k * J->nb + r - ((int64_t)1 << k) + 1]);
                if (v[m] < v[best]) best = m;
            }
            for (int64_t x = bj << AB_SHIFT; x <= j; x++) if (v[x] < v[best]) best = x;
        }
        J->out[t] = best;
    }
    return NULL;
}

EXPORT int oracle_argmin_sparse_blocked(const int64_t *v, int64_t n, const int64_t *qi, const int64_t *qj,
                                        int64_t q, int64_t *out, int threads) {
    if (n <= 0) return q ? -1 : 0;
    int64_t nb = ((n - 1) >> AB_SHIFT) + 1, levels = 1;
    while (((int64_t)1 << levels) <= nb) levels++;
    int64_t *tab = xcalloc((size_t)(nb * levels), sizeof(int64_t));
    for (int64_t b = 0; b < nb; b++) {
        int64_t best = b << AB_SHIFT;
        for (int64_t x = best + 1; x < n && x < ((b + 1) << AB_SHIFT); x++) if (v[x] < v[best]) best = x;
        tab[b] = best;
    }
    for (int64_t k = 1; k < levels; k++)
        for (int64_t b = 0; b + ((int64_t)1 << k) <= nb; b++)
            tab[k * nb + b] = ab_pick(v, tab[(k - 1) * nb + b], tab[(k - 1) * nb + b + ((int64_t)1 << (k - 1))]);
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    ArgminJob jobs[256];
    for (int w = 0; w < threads; w++) {
        jobs[w] = (ArgminJob){v, qi, qj, NULL, tab, n, nb, q * w / threads, q * (w + 1) / threads, out, 0};
        pthread_create(&th[w], NULL, argmin_worker, &jobs[w]);
    }
    int bad = 0;
    for (int w = 0; w < threads; w++) {
        pthread_join(th[w], NULL);
        bad |= jobs[w].bad;
    }
    free(tab);
    return bad ? -1 : 0;
}

/* ------------------------------------------------------------------ */
/* Longest overlap via the generalized suffix array (overlap.py:72-152) */
/* ------------------------------------------------------------------ */

/* encode (sequence.py:144-157) shifted by one, separator rank 1
 * (GeneralizedText.build, overlap.py:83-95).  Returns sigma, or -(1+pos)
 * of the first illegal residue (pos counted in A then B as A-pos / n_a+B-pos). */
static int64_t build_gsa(const uint8_t *a, int64_t na, const uint8_t *b, int64_t nb,
                         int keep_n, int32_t *out) {
    int32_t lut[256];
    memset(lut, 0, sizeof(lut));
    lut['A'] = 1; lut['C'] = 2; lut['G'] = 3; lut['T'] = 4;
    if (keep_n) lut['N'] = 5;
    for (int64_t i = 0; i < na; i++) {
        int32_t r = lut[a[i]];
        if (!r) return -(1 + i);
        out[i] = r + 1;
    }
    out[na] = 1;
    for (int64_t i = 0; i < nb; i++) {
        int32_t r = lut[b[i]];
        if (!r) return -(1 + na + i);
        out[na + 1 + i] = r + 1;
    }
    return (keep_n ? 5 : 4) + 1;
}

/* longest_overlap (overlap.py:110-152).  out = {length, pos_a, pos_b}.
 * Returns 0, or -(1+pos) for an illegal residue at GSA-relative pos. */
EXPORT int64_t oracle_longest_overlap(const uint8_t *a, int64_t na,
                                      const uint8_t *b, int64_t nb, int keep_n,
                                      int64_t *out) {
    out[0] = out[1] = out[2] = 0;
    if (na == 0 || nb == 0) return 0;
    int64_t n = na + nb + 1;
    int32_t *t = xcalloc((size_t)n, sizeof(int32_t));
    int64_t sigma = build_gsa(a, na, b, nb, keep_n, t);
    if (sigma < 0) { free(t); return sigma; }
    int64_t *sa = xcalloc((size_t)n, sizeof(int64_t));
    int64_t *rank = xcalloc((size_t)n, sizeof(int64_t));
    int64_t *lcp = xcalloc((size_t)n, sizeof(int64_t));
    oracle_dc3(t, n, sigma, sa, rank, NULL);
    oracle_lcp(t, n, sa, rank, lcp);
    int64_t boundary = na;
    /* side / cross / best (129-136) */
    int64_t best = -1;
    for (int64_t i = 1; i < n; i++) {
        int64_t p = sa[i - 1], q = sa[i];
        int sp = p < boundary ? 0 : (p > boundary ? 1 : -1);
        int sq = q < boundary ? 0 : (q > boundary ? 1 : -1);
        if (sp >= 0 && sq >= 0 && sp != sq && lcp[i] > best) best = lcp[i];
    }
    if (best <= 0) goto done;
    /* runs of lcp >= best; per-run min A/B position; lexicographic min (138-152) */
    {
        int64_t best_a = INT64_MAX, best_b = INT64_MAX;
        int64_t run_a = INT64_MAX, run_b = INT64_MAX;
        for (int64_t i = 0; i <= n; i++) {
            if (i == n || (i > 0 && lcp[i] < best)) {
                if (run_a != INT64_MAX && run_b != INT64_MAX &&
                    (run_a < best_a || (run_a == best_a && run_b < best_b))) {
                    best_a = run_a;
                    best_b = run_b;
                }
                run_a = run_b = INT64_MAX;
                if (i == n) break;
            }
            int64_t p = sa[i];
            if (p < boundary) { if (p < run_a) run_a = p; }
            else if (p > boundary) { if (p < run_b) run_b = p; }
        }
        out[0] = best;
        out[1] = best_a;
        out[2] = best_b - boundary - 1;
    }
done:
    free(t); free(sa); free(rank); free(lcp);
    return 0;
}

/* Batched pairs across host threads: pair p is A = seqs[offs[2p]..offs[2p+1]),
 * B = seqs[offs[2p+1]..offs[2p+2]).  out is npairs x 3. */
typedef struct {
    const uint8_t *seqs;
    const int64_t *offs;
    int64_t lo, hi;
    int keep_n;
    int64_t *out;
    int64_t status;
} batch_job;

static void *batch_worker(void *arg) {
    batch_job *j = arg;
    for (int64_t p = j->lo; p < j->hi; p++) {
        const uint8_t *a = j->seqs + j->offs[2 * p];
        int64_t na = j->offs[2 * p + 1] - j->offs[2 * p];
        const uint8_t *b = j->seqs + j->offs[2 * p + 1];
        int64_t nb = j->offs[2 * p + 2] - j->offs[2 * p + 1];
        int64_t st = oracle_longest_overlap(a, na, b, nb, j->keep_n, j->out + 3 * p);
        if (st && !j->status) j->status = st;
    }
    return NULL;
}

EXPORT int64_t oracle_overlap_batch(const uint8_t *seqs, const int64_t *offs,
                                    int64_t npairs, int keep_n, int64_t *out,
                                    int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 1024) nthreads = 1024;
    pthread_t th[1024];
    batch_job jobs[1024];
    for (int w = 0; w < nthreads; w++) {
        jobs[w] = (batch_job){seqs, offs, npairs * w / nthreads,
                              npairs * (w + 1) / nthreads, keep_n, out, 0};
        pthread_create(&th[w], NULL, batch_worker, &jobs[w]);
    }
    int64_t st = 0;
    for (int w = 0; w < nthreads; w++) {
        pthread_join(th[w], NULL);
        if (jobs[w].status && !st) st = jobs[w].status;
    }
    return st;
}

/* ------------------------------------------------------------------ FASTA */
/* parse_fasta (sequence.py:77-125) for a str source, followed by encode
 * (sequence.py:144-157) when as_ranks: io.StringIO yields lines ending at
 * '\n'; each line is str.strip()-ed (ASCII whitespace \t\n\v\f\r, \x1c-\x1f,
 * space); blank lines skipped; '>' opens a record (header = rest, stripped);
 * other lines need a header first, are upper-cased and every char must be in
 * ACGT (+N).  The loop stops at the first error like the reference's raise.
 * Outputs: res (residues, <= B bytes), rec_start[r] (residue offset of record
 * r; rec_start[nrec] = total), hdr_start / hdr_len (header text in d),
 * counts = {residues, records}; err = {pos, line (0-based), kind (1 empty
 * header, 2 sequence line), line start, headers before} or err[0] = -1. */
static int fa_ws(uint8_t c) { return c == 32 || (c >= 9 && c <= 13) || (c >= 28 && c <= 31); }

EXPORT int oracle_fasta(const uint8_t *d, int64_t B, int keep_n, int as_ranks, uint8_t *res,
                        int64_t *rec_start, int64_t *hdr_start, int64_t *hdr_len, int64_t *counts,
                        int64_t *err) {
    int64_t nres = 0, nrec = 0, line = 0, s = 0;
    err[0] = -1;
    while (s < B) {
        int64_t e = s;
        while (e < B && d[e] != '\n') e++;
        int64_t next = e < B ? e + 1 : B;
        int64_t a = s, z = e;
        while (a < z && fa_ws(d[a])) a++;
        while (z > a && fa_ws(d[z - 1])) z--;
        if (a < z) {
            if (d[a] == '>') {
                int64_t h = a + 1;
                while (h < z && fa_ws(d[h])) h++;
                if (h == z) {
                    err[0] = a; err[1] = line; err[2] = 1; err[3] = a; err[4] = nrec;
                    break;
                }
                rec_start[nrec] = nres;
                hdr_start[nrec] = h;
                hdr_len[nrec] = z - h;
                nrec++;
            } else {
                if (nrec == 0) {
                    err[0] = a; err[1] = line; err[2] = 2; err[3] = a; err[4] = 0;
                    break;
                }
                int bad = 0;
                for (int64_t j = a; j < z; j++) {
                    uint8_t u = d[j];
                    if (u >= 'a' && u <= 'z') u -= 32;
                    int r = u == 'A' ? 1 : u == 'C' ? 2 : u == 'G' ? 3 : u == 'T' ? 4 : (u == 'N' && keep_n) ? 5 : 0;
                    if (!r) {
                        err[0] = j; err[1] = line; err[2] = 2; err[3] = a; err[4] = nrec;
                        bad = 1;
                        break;
                    }
                    res[nres++] = as_ranks ? (uint8_t)r : u;
                }
                if (bad) break;
            }
        }
        line++;
        s = next;
    }
    rec_start[nrec] = nres;
    counts[0] = nres;
    counts[1] = nrec;
    return err[0] >= 0;
}

/* --------------------------------------------------- Cartesian tree / tour */
/* build_cartesian (rmq.py:91-117: rightmost-spine stack, pop while the top is
 * greater) and euler_tour (rmq.py:120-152: iterative DFS emitting a node on
 * entry and after each child returns). */
EXPORT int oracle_cartesian(const int64_t *v, int64_t n, int64_t *parent, int64_t *left, int64_t *right,
                            int64_t *root, int64_t *nodes, int64_t *depths, int64_t *first) {
    if (n <= 0) return -1;
    int64_t *stack = (int64_t *)xcalloc((size_t)n, sizeof(int64_t));
    int64_t top = 0;
    for (int64_t i = 0; i < n; i++) {
        parent[i] = left[i] = right[i] = -1;
    }
    for (int64_t i = 0; i < n; i++) {
        int64_t last = -1;
        while (top > 0 && v[stack[top - 1]] > v[i]) last = stack[--top];
        if (last != -1) {
            left[i] = last;
            parent[last] = i;
        }
        if (top > 0) {
            right[stack[top - 1]] = i;
            parent[i] = stack[top - 1];
        }
        stack[top++] = i;
    }
    *root = stack[0];
    /* DFS: (node, depth, phase) */
    int64_t *sn = (int64_t *)xcalloc((size_t)(2 * n + 2), sizeof(int64_t));
    int64_t *sd = (int64_t *)xcalloc((size_t)(2 * n + 2), sizeof(int64_t));
    int8_t *sp = (int8_t *)xcalloc((size_t)(2 * n + 2), 1);
    for (int64_t i = 0; i < n; i++) first[i] = -1;
    int64_t sz = 0, pos = 0;
    sn[sz] = *root; sd[sz] = 0; sp[sz] = 0; sz++;
    while (sz > 0) {
        sz--;
        int64_t node = sn[sz], depth = sd[sz];
        int phase = sp[sz];
        nodes[pos] = node;
        depths[pos] = depth;
        if (first[node] < 0) first[node] = pos;
        pos++;
        if (phase == 0) {
            if (left[node] >= 0) {
                sn[sz] = node; sd[sz] = depth; sp[sz] = 1; sz++;
                sn[sz] = left[node]; sd[sz] = depth + 1; sp[sz] = 0; sz++;
                continue;
            }
            phase = 1;
        }
        if (phase == 1 && right[node] >= 0) {
            sn[sz] = node; sd[sz] = depth; sp[sz] = 2; sz++;
            sn[sz] = right[node]; sd[sz] = depth + 1; sp[sz] = 0; sz++;
        }
    }
    free(stack); free(sn); free(sd); free(sp);
    return pos == 2 * n - 1 ? 0 : -2;
}
