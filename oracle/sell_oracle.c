/*
 * sell_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded CPU restatement of the reference `sellkit`
 * SELL-C-sigma build and multiplication kernels.  It is the checker for the
 * CUDA product path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  The product library
 * (libsellb200.so) never links or calls it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/sellkit and
 * the reference's own compiled Cython core built by oracle/build_ref.sh).
 *
 * Compile with -ffp-contract=off: the reference's compiled core contains no
 * FMA (every product and sum is separately rounded), and neither may this.
 *
 * Status codes: 0 ok, -1 parameter error (mirrors sellkit ParameterError).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* sigma resolution: formats.py:321-334                                    */
/* ---------------------------------------------------------------------- */

/* Returns sigma_eff (>=1) or -1 when sigma is not a multiple of C inside
 * (C, n_rows).  n_pad = ceil(n/C)*C (formats.py:322). */
int64_t oracle_sigma_eff(int64_t n_rows, int64_t C, int64_t sigma)
{
    if (C < 1 || sigma < 1) return -1;
    int64_t n_pad = n_rows ? ((n_rows + C - 1) / C) * C : 0;
    if (sigma <= C) return 1;                      /* formats.py:325-328 */
    if (sigma >= n_rows) return n_pad > 1 ? n_pad : 1;
    if (sigma % C != 0) return -1;                 /* formats.py:329-332 */
    return sigma;
}

/* ---------------------------------------------------------------------- */
/* _scope_order: formats.py:285-292 (lexsort keys: scope asc, len desc,    */
/* original index asc).  Stable merge sort per scope on (len desc, idx).   */
/* ---------------------------------------------------------------------- */

static void merge_desc(int64_t *a, int64_t *tmp, int64_t lo, int64_t mid,
                       int64_t hi, const int64_t *len)
{
    int64_t i = lo, j = mid, k = lo;
    while (i < mid && j < hi) {
        /* take from the right only if strictly longer: keeps index order on ties */
        if (len[a[j]] > len[a[i]]) tmp[k++] = a[j++];
        else tmp[k++] = a[i++];
    }
    while (i < mid) tmp[k++] = a[i++];
    while (j < hi) tmp[k++] = a[j++];
    memcpy(a + lo, tmp + lo, (size_t)(hi - lo) * sizeof(int64_t));
}

static void msort_desc(int64_t *a, int64_t *tmp, int64_t lo, int64_t hi,
                       const int64_t *len)
{
    if (hi - lo < 2) return;
    int64_t mid = lo + (hi - lo) / 2;
    msort_desc(a, tmp, lo, mid, len);
    msort_desc(a, tmp, mid, hi, len);
    if (len[a[mid - 1]] >= len[a[mid]]) return;    /* already ordered */
    merge_desc(a, tmp, lo, mid, hi, len);
}

static int64_t gcd64(int64_t a, int64_t b)
{
    while (b) { int64_t t = a % b; a = b; b = t; }
    return a;
}

/*
 * Phase 1 of crs_to_sell (formats.py:309-360): parameter checks, sigma
 * resolution, scope order, perm, row_lengths, cl (with align rounding) and cs.
 * Output buffers: order[n_pad] (stored row p holds padded original row
 * order[p]), perm[n_rows], row_lengths[n_pad], cl[n_chunks], cs[n_chunks+1].
 * n_pad = ceil(n/C)*C, n_chunks = n_pad/C (caller computes them the same way).
 */
int oracle_sell_plan(const int64_t *rpt, int64_t n_rows, int64_t C,
                     int64_t sigma, int64_t align_bytes,
                     int64_t *order, int32_t *perm, int32_t *row_lengths,
                     int32_t *cl, int64_t *cs)
{
    if (C < 1 || sigma < 1) return -1;                  /* formats.py:309-312 */
    if (align_bytes != 1 && align_bytes != 64) return -1; /* :313-314 */
    int64_t sigma_eff = oracle_sigma_eff(n_rows, C, sigma);
    if (sigma_eff < 0) return -1;
    int64_t n = n_rows;
    int64_t n_pad = n ? ((n + C - 1) / C) * C : 0;
    int64_t n_chunks = n_pad / C;

    int64_t *len = (int64_t *)malloc((size_t)(n_pad ? n_pad : 1) * sizeof(int64_t));
    if (!len) return -4;
    for (int64_t p = 0; p < n_pad; ++p)                 /* formats.py:336-338 */
        len[p] = p < n ? rpt[p + 1] - rpt[p] : 0;

    for (int64_t p = 0; p < n_pad; ++p) order[p] = p;
    if (sigma_eff > 1) {                                /* formats.py:344-349 */
        int64_t *tmp = (int64_t *)malloc((size_t)n_pad * sizeof(int64_t));
        if (!tmp) { free(len); return -4; }
        for (int64_t s0 = 0; s0 < n_pad; s0 += sigma_eff) {
            int64_t s1 = s0 + sigma_eff < n_pad ? s0 + sigma_eff : n_pad;
            msort_desc(order, tmp, s0, s1, len);
        }
        free(tmp);
    }
    for (int64_t p = 0; p < n_pad; ++p) {
        if (order[p] < n) perm[order[p]] = (int32_t)p;  /* perm_full[order]=arange */
        row_lengths[p] = (int32_t)len[order[p]];        /* sorted_len */
    }

    int64_t unit = 1;                                   /* formats.py:352-356 */
    if (align_bytes > 1) unit = align_bytes / gcd64(4 * C, align_bytes);
    cs[0] = 0;
    for (int64_t c = 0; c < n_chunks; ++c) {            /* formats.py:351,358-360 */
        int64_t m = 0;
        for (int64_t r = 0; r < C; ++r) {
            int64_t l = row_lengths[c * C + r];
            if (l > m) m = l;
        }
        if (unit > 1) m = ((m + unit - 1) / unit) * unit;
        cl[c] = (int32_t)m;
        cs[c + 1] = cs[c] + C * m;
    }
    free(len);
    return 0;
}

/*
 * Phase 2 (formats.py:362-377): zero-filled val/col of cs[n_chunks] slots,
 * then scatter of row p's j-th entry to cs[p/C] + j*C + p%C.  With
 * permute_cols the column index is mapped through perm.
 */
int oracle_sell_fill(const int64_t *rpt, const int32_t *col_in,
                     const double *val_in, int64_t n_rows, int64_t C,
                     const int64_t *order, const int32_t *perm,
                     const int32_t *row_lengths, const int64_t *cs,
                     int permute_cols, int32_t *col_out, double *val_out)
{
    int64_t n_pad = n_rows ? ((n_rows + C - 1) / C) * C : 0;
    int64_t n_chunks = n_pad / C;
    int64_t total = cs[n_chunks];
    memset(col_out, 0, (size_t)total * sizeof(int32_t));
    memset(val_out, 0, (size_t)total * sizeof(double));
    for (int64_t p = 0; p < n_pad; ++p) {
        int64_t o = order[p];
        if (o >= n_rows) continue;                      /* padding row, len 0 */
        int64_t src = rpt[o];
        int64_t dst = cs[p / C] + p % C;
        for (int64_t j = 0; j < row_lengths[p]; ++j) {
            int32_t c = col_in[src + j];
            val_out[dst + j * C] = val_in[src + j];
            col_out[dst + j * C] = permute_cols ? perm[c] : c;
        }
    }
    return 0;
}

/* fp32 flavour of the fill (values moved, never rounded). */
int oracle_sell_fill_f32(const int64_t *rpt, const int32_t *col_in,
                         const float *val_in, int64_t n_rows, int64_t C,
                         const int64_t *order, const int32_t *perm,
                         const int32_t *row_lengths, const int64_t *cs,
                         int permute_cols, int32_t *col_out, float *val_out)
{
    int64_t n_pad = n_rows ? ((n_rows + C - 1) / C) * C : 0;
    int64_t n_chunks = n_pad / C;
    int64_t total = cs[n_chunks];
    memset(col_out, 0, (size_t)total * sizeof(int32_t));
    memset(val_out, 0, (size_t)total * sizeof(float));
    for (int64_t p = 0; p < n_pad; ++p) {
        int64_t o = order[p];
        if (o >= n_rows) continue;
        int64_t src = rpt[o];
        int64_t dst = cs[p / C] + p % C;
        for (int64_t j = 0; j < row_lengths[p]; ++j) {
            int32_t c = col_in[src + j];
            val_out[dst + j * C] = val_in[src + j];
            col_out[dst + j * C] = permute_cols ? perm[c] : c;
        }
    }
    return 0;
}

/* ---------------------------------------------------------------------- */
/* Kernels: _kernels.pyx                                                   */
/* ---------------------------------------------------------------------- */

/* spmv_sell_range, _kernels.pyx:65-92: per chunk, C running sums from +0.0,
 * slot order, padding included, y stored or accumulated once per row. */
int oracle_spmv_sell_range(const int64_t *cs, const int32_t *cl, int64_t C,
                           const int32_t *col, const double *val,
                           const double *x, double *y, int64_t c0, int64_t c1,
                           int accumulate)
{
    double *tmp = (double *)malloc((size_t)C * sizeof(double));
    if (!tmp) return -4;
    for (int64_t i = c0; i < c1; ++i) {
        for (int64_t r = 0; r < C; ++r) tmp[r] = 0.0;
        int64_t flat = cs[i];
        for (int64_t j = 0; j < cl[i]; ++j) {
            for (int64_t r = 0; r < C; ++r)
                tmp[r] = tmp[r] + val[flat + r] * x[col[flat + r]];
            flat += C;
        }
        int64_t row0 = i * C;
        if (accumulate)
            for (int64_t r = 0; r < C; ++r) y[row0 + r] = y[row0 + r] + tmp[r];
        else
            for (int64_t r = 0; r < C; ++r) y[row0 + r] = tmp[r];
    }
    free(tmp);
    return 0;
}

/* Same loop in binary32 arithmetic (no reference path exists for fp32; the
 * reference is fp64-only, formats.py:18).  Used for bitwise fp32 parity. */
int oracle_spmv_sell_range_f32(const int64_t *cs, const int32_t *cl, int64_t C,
                               const int32_t *col, const float *val,
                               const float *x, float *y, int64_t c0, int64_t c1,
                               int accumulate)
{
    float *tmp = (float *)malloc((size_t)C * sizeof(float));
    if (!tmp) return -4;
    for (int64_t i = c0; i < c1; ++i) {
        for (int64_t r = 0; r < C; ++r) tmp[r] = 0.0f;
        int64_t flat = cs[i];
        for (int64_t j = 0; j < cl[i]; ++j) {
            for (int64_t r = 0; r < C; ++r)
                tmp[r] = tmp[r] + val[flat + r] * x[col[flat + r]];
            flat += C;
        }
        int64_t row0 = i * C;
        if (accumulate)
            for (int64_t r = 0; r < C; ++r) y[row0 + r] = y[row0 + r] + tmp[r];
        else
            for (int64_t r = 0; r < C; ++r) y[row0 + r] = tmp[r];
    }
    free(tmp);
    return 0;
}

/* spmv_crs_range, _kernels.pyx:17-31 */
int oracle_spmv_crs_range(const int64_t *rpt, const int32_t *col,
                          const double *val, const double *x, double *y,
                          int64_t r0, int64_t r1, int accumulate)
{
    for (int64_t i = r0; i < r1; ++i) {
        double tmp = 0.0;
        for (int64_t j = rpt[i]; j < rpt[i + 1]; ++j)
            tmp = tmp + val[j] * x[col[j]];
        y[i] = accumulate ? y[i] + tmp : tmp;
    }
    return 0;
}

/* spmv_crs_unrolled_range, _kernels.pyx:34-62: four partial sums over the
 * multiple-of-4 prefix, combined ((t0+t1)+t2)+t3 (after y when accumulating),
 * then the remainder loop. */
int oracle_spmv_crs_unrolled_range(const int64_t *rpt, const int32_t *col,
                                   const double *val, const double *x,
                                   double *y, int64_t r0, int64_t r1,
                                   int accumulate)
{
    for (int64_t i = r0; i < r1; ++i) {
        int64_t s = rpt[i], e = rpt[i + 1];
        int64_t m = s + ((e - s) & ~(int64_t)3);
        double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0, acc;
        int64_t j = s;
        while (j < m) {
            t0 = t0 + val[j] * x[col[j]];
            t1 = t1 + val[j + 1] * x[col[j + 1]];
            t2 = t2 + val[j + 2] * x[col[j + 2]];
            t3 = t3 + val[j + 3] * x[col[j + 3]];
            j += 4;
        }
        if (accumulate) acc = y[i] + (((t0 + t1) + t2) + t3);
        else acc = ((t0 + t1) + t2) + t3;
        while (j < e) { acc = acc + val[j] * x[col[j]]; ++j; }
        y[i] = acc;
    }
    return 0;
}

/* read_sum, _kernels.pyx:142-161: eight strided partial sums + remainder. */
double oracle_read_sum(const double *a, int64_t n)
{
    int64_t i = 0, n8 = n - (n % 8);
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0, s7 = 0;
    double rest = 0;
    while (i < n8) {
        s0 += a[i]; s1 += a[i + 1]; s2 += a[i + 2]; s3 += a[i + 3];
        s4 += a[i + 4]; s5 += a[i + 5]; s6 += a[i + 6]; s7 += a[i + 7];
        i += 8;
    }
    while (i < n) { rest += a[i]; ++i; }
    return (((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7))) + rest;
}

/* ---------------------------------------------------------------------- */
/* canonicalize_coo + coo_to_crs: formats.py:89-108, 169-175.              */
/* Order: np.lexsort((cols, rows)) = stable sort by (row, col).  Runs of   */
/* equal coordinates are summed like np.add.reduceat: the run's first      */
/* value plus NumPy's pairwise_sum of the rest (restated below: < 8 terms  */
/* sequentially from -0.0; <= 128 terms in eight interleaved partial sums, */
/* combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail; longer     */
/* runs split at n/2 rounded down to a multiple of 8).                     */
/* ---------------------------------------------------------------------- */

static const int64_t *g_r, *g_c;   /* sort keys (single-threaded oracle) */

static int key_less(int64_t a, int64_t b)
{
    return g_r[a] < g_r[b] || (g_r[a] == g_r[b] && g_c[a] < g_c[b]);
}

static void msort_key(int64_t *a, int64_t *tmp, int64_t lo, int64_t hi)
{
    if (hi - lo < 2) return;
    int64_t mid = lo + (hi - lo) / 2;
    msort_key(a, tmp, lo, mid);
    msort_key(a, tmp, mid, hi);
    int64_t i = lo, j = mid, k = lo;
    while (i < mid && j < hi) tmp[k++] = key_less(a[j], a[i]) ? a[j++] : a[i++];
    while (i < mid) tmp[k++] = a[i++];
    while (j < hi) tmp[k++] = a[j++];
    memcpy(a + lo, tmp + lo, (size_t)(hi - lo) * sizeof(int64_t));
}

static double np_pairwise(const double *v, const int64_t *ord, int64_t n)
{
    if (n < 8) {
        double r = -0.0;
        for (int64_t i = 0; i < n; ++i) r += v[ord[i]];
        return r;
    }
    if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; ++j) r[j] = v[ord[j]];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += v[ord[i + j]];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += v[ord[i]];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise(v, ord, n2) + np_pairwise(v, ord + n2, n - n2);
}

/* Inputs must be in bounds (the COOMatrix constructor checks).  Writes rpt
 * [n_rows+1], col/val [<= nnz]; returns the canonical nnz, or -1. */
int64_t oracle_coo_to_crs(const int64_t *rows, const int64_t *cols, const double *vals,
                          int64_t nnz, int64_t n_rows, int64_t *rpt, int32_t *col,
                          double *val)
{
    int64_t *ord = malloc((size_t)(nnz ? nnz : 1) * sizeof(int64_t));
    int64_t *tmp = malloc((size_t)(nnz ? nnz : 1) * sizeof(int64_t));
    if (!ord || !tmp) { free(ord); free(tmp); return -1; }
    for (int64_t i = 0; i < nnz; ++i) ord[i] = i;
    g_r = rows; g_c = cols;
    msort_key(ord, tmp, 0, nnz);
    int64_t u = 0;
    for (int64_t s = 0; s < nnz;) {
        int64_t e = s + 1;
        while (e < nnz && rows[ord[e]] == rows[ord[s]] && cols[ord[e]] == cols[ord[s]]) ++e;
        double v = vals[ord[s]];
        if (e - s > 1) v = v + np_pairwise(vals, ord + s + 1, e - s - 1);
        col[u] = (int32_t)cols[ord[s]];
        val[u] = v;
        tmp[u] = rows[ord[s]];          /* row of unique entry u */
        ++u;
        s = e;
    }
    /* rpt = cumsum(bincount(rows, minlength=n_rows)), formats.py:171-173 */
    for (int64_t r = 0; r <= n_rows; ++r) rpt[r] = 0;
    for (int64_t k = 0; k < u; ++k) rpt[tmp[k] + 1] += 1;
    for (int64_t r = 0; r < n_rows; ++r) rpt[r + 1] += rpt[r];
    free(ord); free(tmp);
    return u;
}

/* ---------------------------------------------------------------------- */
/* LRU replay of a line-id stream: _kernels.pyx:95-139 (cachesim.py:74)    */
/* ---------------------------------------------------------------------- */

/* Fully-associative LRU cache of cache_lines lines, replayed access by
 * access with an intrusive doubly-linked recency list over the dense id
 * table (two sentinels after the n_slots ids).  Returns the miss count, or
 * -1 when memory runs out. */
int64_t oracle_lru_stream_misses(const int64_t *lines, int64_t n, int64_t cache_lines,
                                 int64_t n_slots)
{
    if (n == 0) return 0;
    if (cache_lines <= 0) return n;
    const int64_t mru = n_slots, lru = n_slots + 1;       /* sentinels */
    int64_t *fwd = malloc((size_t)(n_slots + 2) * sizeof(int64_t));   /* toward LRU */
    int64_t *bwd = malloc((size_t)(n_slots + 2) * sizeof(int64_t));   /* toward MRU */
    unsigned char *in = calloc((size_t)(n_slots ? n_slots : 1), 1);
    if (!fwd || !bwd || !in) { free(fwd); free(bwd); free(in); return -1; }
    fwd[mru] = lru;
    bwd[lru] = mru;
    int64_t misses = 0, held = 0;
    for (int64_t k = 0; k < n; ++k) {
        const int64_t l = lines[k];
        if (in[l]) {                       /* hit: detach, re-attach at MRU */
            fwd[bwd[l]] = fwd[l];
            bwd[fwd[l]] = bwd[l];
        } else {
            ++misses;
            if (held == cache_lines) {     /* evict the least recent line */
                const int64_t v = bwd[lru];
                fwd[bwd[v]] = lru;
                bwd[lru] = bwd[v];
                in[v] = 0;
            } else {
                ++held;
            }
            in[l] = 1;
        }
        fwd[l] = fwd[mru];
        bwd[fwd[mru]] = l;
        bwd[l] = mru;
        fwd[mru] = l;
    }
    free(fwd); free(bwd); free(in);
    return misses;
}
