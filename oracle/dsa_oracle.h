/*
 * dsa_oracle.h -- CPU restatement of the reference DSA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker for the sm_100a
 * kernels in paper_2110_11299_b200/; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It is
 * never linked into, or called by, the product path.
 *
 * Parity pin: every function below is cross-checked bit-for-bit against the
 * reference implementation compiled from /root/reference/proj/src into
 * oracle/_ref/libdsattn_ref.so (see oracle/Makefile and
 * tests/test_oracle_vs_reference.py), and against golden vectors generated
 * from that library (tests/golden/, oracle/gen_golden.py).
 *
 * Reference anchors (P/ = /root/reference/proj/):
 *   projection     P/src/kernels/scalar.cpp:19-32 (sequential FMA, ascending k)
 *                  P/src/linalg.cpp:11-17 (f32 rounding of the product)
 *   quantize       P/src/predictor.cpp:34-45, P/src/kernels/scalar.cpp:11-17,60-68
 *   row top-k      P/src/linalg.cpp:69-85 (value desc, index asc; output asc)
 *   colvec         P/src/maskgen.cpp:33-61 (band structure; max-pool extension)
 *   threshold      P/src/maskgen.cpp:22-31 (>= theta; causal/fixed-point ext.)
 *   sddmm          P/src/sparse.cpp:38-53, P/src/kernels/scalar.cpp:34-45
 *   sparse softmax P/src/sparse.cpp:55-78 (empty row -> zero, flagged)
 *   spmm           P/src/sparse.cpp:80-91, P/src/kernels/scalar.cpp:47-58
 */
#ifndef DSA_ORACLE_H
#define DSA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* x[L x k] = q[L x d] . p[d x k]; per element acc = fma(q[i][t], p[t][j], acc)
 * for t ascending from acc = 0 (scalar.cpp:19-32).  round_f32 != 0 rounds each
 * result through float, as linalg.cpp:15 does when both operands are f32. */
void dsa_oracle_project(const double* q, const double* p, int64_t L, int64_t d, int64_t k,
                        int round_f32, double* x);

/* round half away from zero, operation for operation (scalar.cpp:11-17). */
double dsa_oracle_round_half_away(double x);

/* Per-tensor symmetric quantisation (predictor.cpp:34-45): amax = max |x|,
 * s = amax / qmax, level = clamp(round_half_away(x / s), +-qmax).  Writes the
 * integer levels; returns s (0.0 when amax == 0, all levels 0). */
double dsa_oracle_quantize_levels(const double* x, int64_t n, int bits, int32_t* levels);

/* Same rule applied independently to every row of a rows x cols tensor
 * (per-row extension); scales[r] = amax_r / qmax. */
void dsa_oracle_quantize_levels_rows(const double* x, int64_t rows, int64_t cols, int bits,
                                     int32_t* levels, double* scales);

/* Dequantised values exactly as the reference quantize() returns them:
 * y = level * s, rounded through float when round_f32 (predictor.cpp:43). */
void dsa_oracle_dequantize(const int32_t* levels, int64_t n, double s, int round_f32, double* y);

/* Exact integer approximate scores S[i][j] = <lq_i, lk_j> (L x L, int32). */
void dsa_oracle_scores_int(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k,
                           int32_t* s);

/* Row top-k of one row of doubles with the reference comparator
 * (value desc, then index asc), result ascending (linalg.cpp:69-85).
 * Returns 0, or -1 when keep is outside [1, n] (ParamError). */
int dsa_oracle_row_topk(const double* row, int64_t n, int64_t keep, uint32_t* out);

/* Row-wise top-k mask on exact integer scores (O3): cols[L x keep]. */
int dsa_oracle_mask_topk(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k,
                         int64_t keep, uint32_t* cols);

/* Row-wise top-k on per-row-quantised levels (S5): rank key j of row i by
 * (double)S_int[i][j] * sk[j] (one correctly-rounded multiply). */
int dsa_oracle_mask_topk_rowscaled(const int32_t* lq, const int32_t* lk, const double* sk,
                                   int64_t L, int64_t k, int64_t keep, uint32_t* cols);

/* Vector-wise (v query rows x 1 key column) mask, max-pooled over the band
 * (O4): band b covers rows [b*v, min(b*v+v, L)); band_cols[nb x keep]. */
int dsa_oracle_mask_colvec(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k,
                           int64_t v, int64_t keep, uint32_t* band_cols);

/* Block-wise mask (O5): block score = mean of S_int over the bs x bs block
 * (compared exactly as sum_a * cnt_b vs sum_b * cnt_a), optional forced
 * diagonal, keep_blocks per block-row; block_cols[nbr x keep_blocks]. */
int dsa_oracle_mask_block(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k,
                          int64_t bs, int64_t keep_blocks, int force_diag, uint32_t* block_cols);

/* Deterministic exp used by the threshold rule (Cody-Waite + degree-13
 * Horner, fma only): identical bits on any IEEE-754 fma machine. */
double dsa_oracle_exp(double x);

/* Fixed-point softmax weight table for the threshold rule (O6):
 * E[t] = nearbyint(dsa_exp(c * -t) * 2^40) for t = 0..n-1 (t = M_i - S). */
void dsa_oracle_exp_table(double c, int64_t n, int64_t* E);

/* Threshold mask (O6): per row i over candidates j (j <= i when causal),
 * M_i = max S, Z_i = sum E[M_i - S_ij] (exact int64), keep j iff
 * E[M_i - S_ij] * L * frac_num >= Z_i * frac_den   (p >= frac_den/(frac_num*L)),
 * then at most cap kept (largest S, lowest index).  c = s_q*s_k/sqrt(d).
 * Two-pass interface: call with cols == NULL to get rowptr[L+1] (counts
 * prefix), then with cols sized rowptr[L].  Returns number of empty rows. */
int64_t dsa_oracle_mask_threshold(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k,
                                  double c, int64_t frac_num, int64_t frac_den, int64_t cap,
                                  int causal, uint64_t* rowptr, uint32_t* cols);

/* Sparse attention for one head (O7): sddmm (fma over d ascending, times
 * 1/sqrt(d) when scale) -> two-pass f64 softmax per row (empty row: zero,
 * flagged) -> spmm (fma over kept positions ascending).  round_f32 rounds Z
 * through float (V is an f32 Matrix, sparse.cpp:84-88). */
void dsa_oracle_sparse_attention(const double* q, const double* k, const double* v, int64_t L,
                                 int64_t d, int64_t dv, const uint64_t* rowptr,
                                 const uint32_t* cols, int scale, int round_f32, double* z,
                                 uint8_t* empty_row);

/* Dense additive-mask attention (P/src/attention.cpp:54-71, 99-117): the
 * secondary oracle; -1e4 at masked positions, dense row softmax, A.V. */
void dsa_oracle_masked_dense_attention(const double* q, const double* k, const double* v,
                                       int64_t L, int64_t d, int64_t dv, const uint64_t* rowptr,
                                       const uint32_t* cols, int scale, double* z);

#ifdef __cplusplus
}
#endif
#endif
