/*
 * dsa_oracle.c -- CPU restatement of the reference DSA hot path.
 * TEST INFRASTRUCTURE ONLY (see dsa_oracle.h): the checker, never the product.
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, as P/CMakeLists.txt:13-17).
 */
#include "dsa_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ projection */

/* P/src/kernels/scalar.cpp:19-32: c[i][j] starts at 0 and sees
 * acc = fma(a[i][t], b[t][j], acc) for t = 0..k-1 ascending. */
void dsa_oracle_project(const double* q, const double* p, int64_t L, int64_t d, int64_t k,
                        int round_f32, double* x) {
    for (int64_t i = 0; i < L; ++i) {
        for (int64_t j = 0; j < k; ++j) {
            double acc = 0.0;
            for (int64_t t = 0; t < d; ++t) acc = fma(q[i * d + t], p[t * k + j], acc);
            x[i * k + j] = round_f32 ? (double)(float)acc : acc;
        }
    }
}

/* P/src/kernels/scalar.cpp:11-17 */
double dsa_oracle_round_half_away(double x) {
    double t = trunc(x);
    double f = x - t;
    if (f >= 0.5) t += 1.0;
    if (f <= -0.5) t -= 1.0;
    return t;
}

static double qmax_of(int bits) { return (double)((1 << (bits - 1)) - 1); }

static int32_t level_of(double x, double s, double qmax) {
    /* P/src/kernels/scalar.cpp:60-68 */
    double r = dsa_oracle_round_half_away(x / s);
    if (r > qmax) r = qmax;
    if (r < -qmax) r = -qmax;
    return (int32_t)r;
}

/* P/src/predictor.cpp:34-45 with max_abs from P/src/linalg.cpp:93-97 */
double dsa_oracle_quantize_levels(const double* x, int64_t n, int bits, int32_t* levels) {
    const double qmax = qmax_of(bits);
    double amax = 0.0;
    for (int64_t i = 0; i < n; ++i) amax = fmax(amax, fabs(x[i]));
    if (amax == 0.0) {
        memset(levels, 0, (size_t)n * sizeof(int32_t));
        return 0.0;
    }
    const double s = amax / qmax;
    for (int64_t i = 0; i < n; ++i) levels[i] = level_of(x[i], s, qmax);
    return s;
}

void dsa_oracle_quantize_levels_rows(const double* x, int64_t rows, int64_t cols, int bits,
                                     int32_t* levels, double* scales) {
    for (int64_t r = 0; r < rows; ++r)
        scales[r] = dsa_oracle_quantize_levels(x + r * cols, cols, bits, levels + r * cols);
}

void dsa_oracle_dequantize(const int32_t* levels, int64_t n, double s, int round_f32, double* y) {
    for (int64_t i = 0; i < n; ++i) {
        double v = (double)levels[i] * s;
        y[i] = round_f32 ? (double)(float)v : v;
    }
}

/* ---------------------------------------------------------------- scores */

static inline int32_t dot_i32(const int32_t* a, const int32_t* b, int64_t k) {
    int32_t acc = 0;
    for (int64_t t = 0; t < k; ++t) acc += a[t] * b[t];
    return acc;
}

void dsa_oracle_scores_int(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k,
                           int32_t* s) {
    for (int64_t i = 0; i < L; ++i)
        for (int64_t j = 0; j < L; ++j) s[i * L + j] = dot_i32(lq + i * k, lk + j * k, k);
}

/* ----------------------------------------------------------------- top-k */

/* Reference comparator (P/src/linalg.cpp:77-80): a before b iff
 * row[a] > row[b], or equal values and a < b. */
static inline int before(const double* row, uint32_t a, uint32_t b) {
    if (row[a] != row[b]) return row[a] > row[b];
    return a < b;
}

static void sort_u32(uint32_t* v, int64_t n) {
    /* insertion-merge: small n in practice; use a simple bottom-up merge sort */
    if (n < 2) return;
    uint32_t* tmp = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    for (int64_t w = 1; w < n; w *= 2) {
        for (int64_t lo = 0; lo < n; lo += 2 * w) {
            int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            int64_t a = lo, b = mid, o = lo;
            while (a < mid && b < hi) tmp[o++] = v[a] <= v[b] ? v[a++] : v[b++];
            while (a < mid) tmp[o++] = v[a++];
            while (b < hi) tmp[o++] = v[b++];
        }
        memcpy(v, tmp, (size_t)n * sizeof(uint32_t));
    }
    free(tmp);
}

/* Quickselect on the strict total order `before`, then ascending output. */
int dsa_oracle_row_topk(const double* row, int64_t n, int64_t keep, uint32_t* out) {
    if (keep < 1 || keep > n) return -1;
    uint32_t* idx = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    for (int64_t j = 0; j < n; ++j) idx[j] = (uint32_t)j;
    int64_t lo = 0, hi = n - 1, kth = keep - 1;
    while (lo < hi) {
        uint32_t a = idx[lo], b = idx[(lo + hi) / 2], c = idx[hi], piv;
        /* median of three under `before` */
        if (before(row, a, b)) {
            piv = before(row, b, c) ? b : (before(row, a, c) ? c : a);
        } else {
            piv = before(row, a, c) ? a : (before(row, b, c) ? c : b);
        }
        int64_t i = lo, j = hi;
        while (i <= j) {
            while (before(row, idx[i], piv)) ++i;
            while (before(row, piv, idx[j])) --j;
            if (i <= j) {
                uint32_t t = idx[i];
                idx[i] = idx[j];
                idx[j] = t;
                ++i;
                --j;
            }
        }
        if (kth <= j) hi = j;
        else if (kth >= i) lo = i;
        else break;
    }
    memcpy(out, idx, (size_t)keep * sizeof(uint32_t));
    sort_u32(out, keep);
    free(idx);
    return 0;
}

/* Top-k over integer keys: the same comparator as dsa_oracle_row_topk on
 * the exactly-converted doubles (|key| < 2^53). */
static void topk_int_row(const int64_t* key, int64_t n, int64_t keep, uint32_t* out) {
    double* dk = (double*)malloc((size_t)n * sizeof(double));
    for (int64_t j = 0; j < n; ++j) dk[j] = (double)key[j];
    dsa_oracle_row_topk(dk, n, keep, out);
    free(dk);
}

int dsa_oracle_mask_topk(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k,
                         int64_t keep, uint32_t* cols) {
    if (keep < 1 || keep > L) return -1;
    double* row = (double*)malloc((size_t)L * sizeof(double));
    for (int64_t i = 0; i < L; ++i) {
        for (int64_t j = 0; j < L; ++j) row[j] = (double)dot_i32(lq + i * k, lk + j * k, k);
        dsa_oracle_row_topk(row, L, keep, cols + i * keep);
    }
    free(row);
    return 0;
}

int dsa_oracle_mask_topk_rowscaled(const int32_t* lq, const int32_t* lk, const double* sk,
                                   int64_t L, int64_t k, int64_t keep, uint32_t* cols) {
    if (keep < 1 || keep > L) return -1;
    double* row = (double*)malloc((size_t)L * sizeof(double));
    for (int64_t i = 0; i < L; ++i) {
        for (int64_t j = 0; j < L; ++j)
            row[j] = (double)dot_i32(lq + i * k, lk + j * k, k) * sk[j];
        dsa_oracle_row_topk(row, L, keep, cols + i * keep);
    }
    free(row);
    return 0;
}

/* P/src/maskgen.cpp:33-61 band structure; band score = max over the band's
 * rows of the exact integer score (BASELINE "max-pooled"). */
int dsa_oracle_mask_colvec(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k,
                           int64_t v, int64_t keep, uint32_t* band_cols) {
    if (v < 1 || keep < 1 || keep > L) return -1;
    int64_t* pooled = (int64_t*)malloc((size_t)L * sizeof(int64_t));
    int64_t nb = (L + v - 1) / v;
    for (int64_t b = 0; b < nb; ++b) {
        int64_t r0 = b * v, r1 = r0 + v < L ? r0 + v : L;
        for (int64_t j = 0; j < L; ++j) {
            int64_t m = dot_i32(lq + r0 * k, lk + j * k, k);
            for (int64_t i = r0 + 1; i < r1; ++i) {
                int64_t s = dot_i32(lq + i * k, lk + j * k, k);
                if (s > m) m = s;
            }
            pooled[j] = m;
        }
        topk_int_row(pooled, L, keep, band_cols + b * keep);
    }
    free(pooled);
    return 0;
}

/* Block mean-pooling (O5).  Ranking by mean = sum / count is done exactly
 * by cross-multiplication so ragged edge blocks are compared correctly. */
static int block_before(const int64_t* sum, const int64_t* cnt, int64_t a, int64_t b) {
    /* a before b iff mean_a > mean_b, or equal and a < b */
    __int128 lhs = (__int128)sum[a] * cnt[b], rhs = (__int128)sum[b] * cnt[a];
    if (lhs != rhs) return lhs > rhs;
    return a < b;
}

int dsa_oracle_mask_block(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k,
                          int64_t bs, int64_t keep_blocks, int force_diag, uint32_t* block_cols) {
    int64_t nb = (L + bs - 1) / bs;
    if (bs < 1 || keep_blocks < 1 || keep_blocks > nb) return -1;
    int64_t* sum = (int64_t*)malloc((size_t)nb * sizeof(int64_t));
    int64_t* cnt = (int64_t*)malloc((size_t)nb * sizeof(int64_t));
    uint32_t* sel = (uint32_t*)malloc((size_t)nb * sizeof(uint32_t));
    for (int64_t ib = 0; ib < nb; ++ib) {
        int64_t r0 = ib * bs, r1 = r0 + bs < L ? r0 + bs : L;
        for (int64_t jb = 0; jb < nb; ++jb) {
            int64_t c0 = jb * bs, c1 = c0 + bs < L ? c0 + bs : L, s = 0;
            for (int64_t i = r0; i < r1; ++i)
                for (int64_t j = c0; j < c1; ++j) s += dot_i32(lq + i * k, lk + j * k, k);
            sum[jb] = s;
            cnt[jb] = (r1 - r0) * (c1 - c0);
        }
        /* selection sort of the first keep entries under block_before */
        int64_t nsel = 0;
        if (force_diag) sel[nsel++] = (uint32_t)ib;
        while (nsel < keep_blocks) {
            int64_t best = -1;
            for (int64_t jb = 0; jb < nb; ++jb) {
                int taken = 0;
                for (int64_t t = 0; t < nsel; ++t)
                    if (sel[t] == (uint32_t)jb) taken = 1;
                if (taken) continue;
                if (best < 0 || block_before(sum, cnt, jb, best)) best = jb;
            }
            sel[nsel++] = (uint32_t)best;
        }
        sort_u32(sel, keep_blocks);
        memcpy(block_cols + ib * keep_blocks, sel, (size_t)keep_blocks * sizeof(uint32_t));
    }
    free(sum);
    free(cnt);
    free(sel);
    return 0;
}

/* ------------------------------------------------------------- threshold */

/* Deterministic exp: n = rint(x*log2e); r = x - n*ln2 (two fma steps,
 * Cody-Waite split); e^r by degree-13 Taylor Horner in fma; scale by 2^n.
 * Only IEEE-exact operations (fma, mul, rint, ldexp) are used. */
double dsa_oracle_exp(double x) {
    if (x < -50.0) return 0.0;
    if (x > 50.0) x = 50.0;
    const double log2e = 1.4426950408889634;
    const double ln2_hi = 6.93147180369123816490e-01;
    const double ln2_lo = 1.90821492927058770002e-10;
    double n = rint(x * log2e);
    double r = fma(-n, ln2_hi, x);
    r = fma(-n, ln2_lo, r);
    static const double c[14] = {1.0,
                                 1.0,
                                 0.5,
                                 1.6666666666666666e-01,
                                 4.1666666666666664e-02,
                                 8.3333333333333332e-03,
                                 1.3888888888888889e-03,
                                 1.9841269841269841e-04,
                                 2.4801587301587302e-05,
                                 2.7557319223985893e-06,
                                 2.7557319223985888e-07,
                                 2.5052108385441720e-08,
                                 2.0876756987868100e-09,
                                 1.6059043836821613e-10};
    double p = c[13];
    for (int i = 12; i >= 0; --i) p = fma(p, r, c[i]);
    return ldexp(p, (int)n);
}

void dsa_oracle_exp_table(double c, int64_t n, int64_t* E) {
    for (int64_t t = 0; t < n; ++t) {
        double e = dsa_oracle_exp(c * (double)(-t));
        E[t] = (int64_t)rint(e * 1099511627776.0); /* 2^40 */
    }
}

int64_t dsa_oracle_mask_threshold(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k,
                                  double c, int64_t frac_num, int64_t frac_den, int64_t cap,
                                  int causal, uint64_t* rowptr, uint32_t* cols) {
    int64_t qm = 0;
    for (int64_t i = 0; i < L * k; ++i) {
        int64_t a = lq[i] < 0 ? -lq[i] : lq[i], b = lk[i] < 0 ? -lk[i] : lk[i];
        if (a > qm) qm = a;
        if (b > qm) qm = b;
    }
    const int64_t span = 2 * k * qm * qm + 1; /* max possible M_i - S_ij, plus one */
    int64_t* E = (int64_t*)malloc((size_t)span * sizeof(int64_t));
    dsa_oracle_exp_table(c, span, E);
    int32_t* srow = (int32_t*)malloc((size_t)L * sizeof(int32_t));
    double* keyrow = (double*)malloc((size_t)L * sizeof(double));
    uint32_t* tmp = (uint32_t*)malloc((size_t)L * sizeof(uint32_t));
    int64_t empty = 0;
    uint64_t off = 0;
    if (cols == NULL) rowptr[0] = 0;
    for (int64_t i = 0; i < L; ++i) {
        int64_t n = causal ? i + 1 : L;
        int32_t m = INT32_MIN;
        for (int64_t j = 0; j < n; ++j) {
            srow[j] = dot_i32(lq + i * k, lk + j * k, k);
            if (srow[j] > m) m = srow[j];
        }
        uint64_t z = 0;
        for (int64_t j = 0; j < n; ++j) z += (uint64_t)E[m - srow[j]];
        int64_t cnt = 0;
        for (int64_t j = 0; j < n; ++j) {
            unsigned __int128 lhs = (unsigned __int128)(uint64_t)E[m - srow[j]] * (uint64_t)L *
                                    (uint64_t)frac_num;
            unsigned __int128 rhs = (unsigned __int128)z * (uint64_t)frac_den;
            if (lhs >= rhs) tmp[cnt++] = (uint32_t)j; /* ">= theta", maskgen.cpp:29 */
        }
        if (cnt > cap) {
            for (int64_t t = 0; t < n; ++t) keyrow[t] = -1e300;
            for (int64_t t = 0; t < cnt; ++t) keyrow[tmp[t]] = (double)srow[tmp[t]];
            dsa_oracle_row_topk(keyrow, n, cap, tmp);
            cnt = cap;
        }
        if (cnt == 0) ++empty;
        if (cols == NULL) {
            rowptr[i + 1] = rowptr[i] + (uint64_t)cnt;
        } else {
            memcpy(cols + off, tmp, (size_t)cnt * sizeof(uint32_t));
            off += (uint64_t)cnt;
        }
    }
    free(E);
    free(srow);
    free(keyrow);
    free(tmp);
    return empty;
}

/* ------------------------------------------------------------- attention */

void dsa_oracle_sparse_attention(const double* q, const double* k, const double* v, int64_t L,
                                 int64_t d, int64_t dv, const uint64_t* rowptr,
                                 const uint32_t* cols, int scale, int round_f32, double* z,
                                 uint8_t* empty_row) {
    const double sc = scale ? 1.0 / sqrt((double)d) : 1.0; /* sparse.cpp:48 */
    uint64_t maxrow = 0;
    for (int64_t i = 0; i < L; ++i)
        if (rowptr[i + 1] - rowptr[i] > maxrow) maxrow = rowptr[i + 1] - rowptr[i];
    double* s = (double*)malloc((size_t)(maxrow ? maxrow : 1) * sizeof(double));
    for (int64_t i = 0; i < L; ++i) {
        const uint64_t b = rowptr[i], e = rowptr[i + 1];
        double* zr = z + i * dv;
        for (int64_t c = 0; c < dv; ++c) zr[c] = 0.0;
        if (empty_row) empty_row[i] = (uint8_t)(b == e);
        if (b == e) continue; /* sparse.cpp:63-66, spmm zero row scalar.cpp:51 */
        for (uint64_t p = b; p < e; ++p) { /* sddmm, scalar.cpp:34-45 */
            const double* kr = k + (int64_t)cols[p] * d;
            double acc = 0.0;
            for (int64_t t = 0; t < d; ++t) acc = fma(q[i * d + t], kr[t], acc);
            s[p - b] = acc * sc;
        }
        double m = s[0]; /* sparse.cpp:67-76 */
        for (uint64_t p = 1; p < e - b; ++p) m = fmax(m, s[p]);
        double sum = 0.0;
        for (uint64_t p = 0; p < e - b; ++p) {
            s[p] = exp(s[p] - m);
            sum += s[p];
        }
        for (uint64_t p = 0; p < e - b; ++p) s[p] /= sum;
        for (uint64_t p = b; p < e; ++p) { /* spmm, scalar.cpp:47-58 */
            const double w = s[p - b];
            const double* vr = v + (int64_t)cols[p] * dv;
            for (int64_t c = 0; c < dv; ++c) zr[c] = fma(w, vr[c], zr[c]);
        }
        if (round_f32)
            for (int64_t c = 0; c < dv; ++c) zr[c] = (double)(float)zr[c];
    }
    free(s);
}

void dsa_oracle_masked_dense_attention(const double* q, const double* k, const double* v,
                                       int64_t L, int64_t d, int64_t dv, const uint64_t* rowptr,
                                       const uint32_t* cols, int scale, double* z) {
    const double sc = scale ? 1.0 / sqrt((double)d) : 1.0;
    double* row = (double*)malloc((size_t)L * sizeof(double));
    for (int64_t i = 0; i < L; ++i) {
        uint64_t p = rowptr[i];
        for (int64_t j = 0; j < L; ++j) {
            double acc = 0.0; /* matmul_nt: fma over d ascending (scalar.cpp:19-32) */
            for (int64_t t = 0; t < d; ++t) acc = fma(q[i * d + t], k[j * d + t], acc);
            acc = acc * sc;
            if (p < rowptr[i + 1] && cols[p] == (uint32_t)j) ++p;
            else acc = acc - 1e4; /* attention.cpp:54-71 */
            row[j] = acc;
        }
        double m = row[0]; /* linalg.cpp:51-67 */
        for (int64_t j = 1; j < L; ++j) m = fmax(m, row[j]);
        double sum = 0.0;
        for (int64_t j = 0; j < L; ++j) {
            row[j] = exp(row[j] - m);
            sum += row[j];
        }
        for (int64_t j = 0; j < L; ++j) row[j] /= sum;
        for (int64_t c = 0; c < dv; ++c) {
            double acc = 0.0;
            for (int64_t j = 0; j < L; ++j) acc = fma(row[j], v[j * dv + c], acc);
            z[i * dv + c] = acc;
        }
    }
    free(row);
}
