/*
 * dsa_b200.h -- C-ABI of the B200-native Dynamic Sparse Attention hot path.
 *
 * Plain pointers and sizes only (no torch / C++ types).  All device pointers
 * are caller-owned CUDA global memory; every entry point is stream-ordered
 * and asynchronous on the `stream` it is given (a cudaStream_t passed as
 * void*, NULL = legacy default stream), thread-safe, and allocation-free on
 * the hot path (scratch lives in the caller's workspace).  Errors never
 * cross the boundary as exceptions: each call returns a dsa_status and a
 * thread-local message is kept for dsa_last_error().  The C++ shim
 * (include/dsattn_gpu.hpp) maps the codes back onto the reference exception
 * types (ShapeError / ParamError / ConfigError / IoError; P/include/dsattn/
 * errors.hpp:9-31) so reference callers and CLI exit codes are unchanged.
 *
 * Reference interfaces replaced (P/ = /root/reference/proj/):
 *   dsa_predict_wtilde   <- approx_scores / approx_scores_from_r (R = X P, per-head W~)
 *                           P/include/dsattn/predictor.hpp:44-49, P/src/predictor.cpp:67-80
 *   dsa_predict          <- Matrix quantize(const Matrix&, QuantSpec) applied to
 *                           matmul(Q,P) / matmul(K,P)   P/include/dsattn/predictor.hpp:31-49,
 *                           P/src/predictor.cpp:34-45,67-80; kernels::matmul/quantize
 *                           P/include/dsattn/kernels.hpp:22-35
 *   dsa_select           <- predicted_topk_mask / threshold_mask / colvec_mask
 *                           P/include/dsattn/maskgen.hpp:14-31 (+ block mode)
 *   dsa_sparse_attention <- sddmm -> sparse_softmax -> spmm per head
 *                           P/include/dsattn/sparse.hpp:47-55, P/src/sparse.cpp:38-91
 *   dsa_pipeline         <- the per-head composition above (predict -> select -> attend)
 *   dsa_counters         <- OpCounters P/include/dsattn/sparse.hpp:14-21
 *   dsa_last_error       <- exception what() strings
 *   dsa_project_qkv      <- project_qkv (per-head X W_Q / X W_K / X W_V)
 *                           P/src/attention.cpp:36-46 and the predictor input
 *                           R = X P, P/src/trainer.cpp:162
 */
#ifndef DSA_B200_H
#define DSA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSA_ABI_VERSION 1

typedef enum dsa_status {
    DSA_OK = 0,
    DSA_ERR_SHAPE = 1,   /* ShapeError  (dimension mismatch)          */
    DSA_ERR_PARAM = 2,   /* ParamError  (out-of-range value)          */
    DSA_ERR_CONFIG = 3,  /* ConfigError (bad preset / unknown key)    */
    DSA_ERR_CUDA = 4,    /* CUDA runtime / launch failure             */
    DSA_ERR_IO = 5,      /* IoError                                   */
    DSA_ERR_UNSUPPORTED = 6 /* valid config outside the built kernels */
} dsa_status;

typedef enum dsa_dtype { DSA_F32 = 0, DSA_BF16 = 1 } dsa_dtype;

typedef enum dsa_quant_scope {
    DSA_QUANT_PER_TENSOR = 0, /* reference: one scale per (b,h) tensor, predictor.cpp:37-41 */
    DSA_QUANT_PER_ROW = 1     /* extension: one scale per row of Q~ / K~         */
} dsa_quant_scope;

typedef enum dsa_mask_mode {
    DSA_MASK_ROW_TOPK = 0,  /* keep `keep` keys per query row (maskgen.cpp:11-20)           */
    DSA_MASK_COLVEC = 1,    /* vec_v query rows x 1 key column, max-pooled (maskgen.cpp:33) */
    DSA_MASK_BLOCK = 2,     /* block x block tiles, mean-pooled, optional forced diagonal  */
    DSA_MASK_THRESHOLD = 3  /* p~ >= frac_den / (frac_num * L), optional causal, cap       */
} dsa_mask_mode;

/* One (batch x heads) problem; pairs = batch * heads.  Q/K/V/Z are
 * [pairs][L][d] row-major in `dtype`; P is [d][k] float32. */
typedef struct dsa_config {
    int64_t batch, heads, L, d, k;
    int32_t dtype;        /* dsa_dtype                                           */
    int32_t bits;         /* prediction precision: 2, 4 or 8 (QuantSpec bits)    */
    int32_t quant_scope;  /* dsa_quant_scope                                     */
    int32_t round_proj_f32; /* 1: round Q.P through float (f32 Matrix semantics) */
    int32_t mask_mode;    /* dsa_mask_mode                                       */
    int32_t scale;        /* 1: scores scaled by 1/sqrt(d) (sparse.cpp:48)       */
    int64_t keep;         /* ROW_TOPK: keys/row; COLVEC: columns/band; BLOCK: blocks/block-row */
    int32_t vec_v;        /* COLVEC band height                                  */
    int32_t block;        /* BLOCK tile edge                                     */
    int32_t force_diag;   /* BLOCK: diagonal tile always kept (counts in keep)   */
    int32_t causal;       /* THRESHOLD: candidates j <= i                        */
    int64_t frac_num, frac_den; /* THRESHOLD: theta = frac_den / (frac_num * L)  */
    int64_t cap;          /* THRESHOLD: max kept per row                         */
} dsa_config;

/* Device mask.  Layout by mode (all column lists ascending):
 *   ROW_TOPK : cols[pairs][L][keep]
 *   COLVEC   : cols[pairs][ceil(L/vec_v)][keep]        (shared by the band's rows)
 *   BLOCK    : cols[pairs][ceil(L/block)][keep]        (block-column indices)
 *   THRESHOLD: rowptr[pairs*L + 1] (uint64, global CSR), cols[capacity]
 * empty_rows (optional, uint8[pairs*L]) flags rows with no kept key
 * (sparse.cpp:63-66). */
typedef struct dsa_mask {
    uint32_t* cols;
    uint64_t* rowptr;
    int64_t capacity; /* entries available in cols */
    uint8_t* empty_rows;
} dsa_mask;

typedef struct dsa_counts {
    uint64_t nnz;          /* kept positions over all pairs                */
    uint64_t sddmm_mults;  /* nnz * d   (sparse.cpp:51)                    */
    uint64_t spmm_mults;   /* nnz * d   (sparse.cpp:89)                    */
    uint64_t softmax_exps; /* nnz       (sparse.cpp:75)                    */
    uint64_t empty_rows;
    double flops_predict;  /* 4 L d k per pair                             */
    double flops_score;    /* 2 L^2 k per pair (causal: L(L+1) k)          */
    double flops_attention;/* 4 nnz d                                      */
    double bytes_predict;  /* compulsory HBM bytes per phase */
    double bytes_attention;
} dsa_counts;

/* ----------------------------------------------------------------- meta */
int dsa_abi_version(void);
const char* dsa_last_error(void);
const char* dsa_build_info(void);
dsa_status dsa_config_validate(const dsa_config* cfg);
/* Scratch bytes needed by dsa_predict / dsa_select / dsa_pipeline. */
size_t dsa_workspace_bytes(const dsa_config* cfg);
/* Entries needed in dsa_mask.cols (THRESHOLD: worst case from cap, theta, causal). */
int64_t dsa_mask_capacity(const dsa_config* cfg);

/* ------------------------------------------------------------ hot path */
/* (1) projection + quantisation.  levels_q/levels_k: integer levels held
 * exactly in bf16 (uint16 bits), chunk-planar per pair: [pairs][k/8][L][8]
 * (element (r, c) of a pair at ((c/8)*L + r)*8 + c%8 -- a run of rows of one
 * 8-column chunk is contiguous, which makes tensor-core tiles single bulk
 * copies); scale_q/scale_k: [pairs] (PER_TENSOR) or [pairs][L] (PER_ROW)
 * doubles. */
dsa_status dsa_predict(const dsa_config* cfg, const void* q, const void* k, const float* p,
                       uint16_t* levels_q, uint16_t* levels_k, double* scale_q, double* scale_k,
                       void* workspace, size_t workspace_bytes, void* stream);

/* (1') The reference's own predictor entry point, approx_scores /
 * approx_scores_from_r (P/include/dsattn/predictor.hpp:44-49,
 * P/src/predictor.cpp:67-80) with its trainable per-head k x k W~:
 *     R = X P  (per sample, shared by the heads, P/src/trainer.cpp:162),
 *     Q~[b,h] = quantize(R[b] W~_Q[h]),  K~[b,h] = quantize(R[b] W~_K[h]).
 * Every product is the reference matmul's sequential fp64 FMA chain
 * (P/src/kernels/scalar.cpp:19-32), rounded through float when
 * cfg->round_proj_f32 (f32 Matrices), so levels and scales are bit-exact.
 *   x : [batch][L][d_model] f64, or NULL: then r is the INPUT
 *   p : [d_model][k] f64 (ignored when x == NULL)
 *   r : [batch][L][k] f64, written when x != NULL
 *   wq, wk: [heads][k][k] f64 (row-major: Q~ = R . wq[h])
 * Outputs as dsa_predict for pair = b * heads + h (quant_scope honoured;
 * cfg->d is not used).  Workspace: dsa_predict_wtilde_workspace_bytes(). */
size_t dsa_predict_wtilde_workspace_bytes(const dsa_config* cfg);
dsa_status dsa_predict_wtilde(const dsa_config* cfg, int64_t d_model, const double* x, const double* p,
                              double* r, const double* wq, const double* wk, uint16_t* levels_q,
                              uint16_t* levels_k, double* scale_q, double* scale_k, void* workspace,
                              size_t workspace_bytes, void* stream);

/* (2) exact-integer approximate scores -> mask selection. */
dsa_status dsa_select(const dsa_config* cfg, const uint16_t* levels_q, const uint16_t* levels_k,
                      const double* scale_q, const double* scale_k, const dsa_mask* mask,
                      void* workspace, size_t workspace_bytes, void* stream);

/* (3) SDDMM -> sparse row softmax -> SpMM over the mask; z: [pairs][L][d]
 * in cfg->dtype.  Empty rows give zero output rows, flagged in
 * mask->empty_rows when non-NULL. */
dsa_status dsa_sparse_attention(const dsa_config* cfg, const void* q, const void* k,
                                const void* v, const dsa_mask* mask, void* z, void* stream);

/* (1)->(2)->(3).  mask_out may be NULL (mask kept in the workspace only). */
dsa_status dsa_pipeline(const dsa_config* cfg, const void* q, const void* k, const void* v,
                        const float* p, void* z, const dsa_mask* mask_out, void* workspace,
                        size_t workspace_bytes, void* stream);

/* (0) the step before the path: every head's Q, K, V and the predictor
 * input R = X P of one attention layer in ONE bf16 tensor-core GEMM over X
 * (fp32 accumulation, outputs rounded once).
 *   x: [batch][L][d_model] bf16, d_model % 64 == 0
 *   w: packed weights [heads*(2*dk + dv) + npred][d_model] bf16 (K-major):
 *      row h*dk + c        = column c of W_Q[h]   (h < heads, c < dk)
 *      row heads*dk + ...  = W_K rows, then heads*dv W_V rows, then the
 *      npred rows of P^T (npred <= 32, 0 = no predictor input)
 *   q, k: [batch*heads][L][dk] bf16; v: [batch*heads][L][dv] bf16 -- the
 *      (b,h)-pair layout dsa_predict / dsa_pipeline consume
 *   r: [batch][L][npred] f32 (NULL when npred == 0)
 * dk, dv in {32, 64, 96, 128, ...} (multiples of 32). */
dsa_status dsa_project_qkv(int64_t batch, int64_t L, int64_t d_model, int64_t heads, int64_t dk,
                           int64_t dv, int64_t npred, const void* x, const void* w, void* q,
                           void* k, void* v, float* r, void* stream);

/* 1 when dsa_pipeline runs selection and attention as ONE fused kernel for
 * this config (COLVEC on the tensor-core path), 0 when it runs them as
 * separate phases, -1 for an invalid config.  Introspection for bench.py's
 * roofline attribution; no reference counterpart. */
int dsa_pipeline_fused(const dsa_config* cfg);

/* Kernels launched by this library since load (process-wide, monotonic);
 * bench.py reads it around timed regions. */
uint64_t dsa_launch_counter(void);

/* prediction_accuracy (P/src/maskgen.cpp:94-107) between two device masks
 * of cfg's layout over all pairs: |pred n oracle| / |pred|.  Per-row
 * counts must be equal (ParamError otherwise, as the reference); empty
 * masks are a ParamError.  Synchronises `stream`. */
dsa_status dsa_prediction_accuracy(const dsa_config* cfg, const dsa_mask* pred, const dsa_mask* oracle,
                                   double* accuracy, void* stream);

/* The reference's dataflow fetch-count model on a device mask
 * (dataflow::simulate, P/include/dsattn/dataflow.hpp:14-46,
 * P/src/dataflow.cpp:10-62): second-operand fetches of SDDMM / SpMM under
 * one of three schedules over bands of `band` consecutive rows (1 <= band
 * <= 32; row_by_row always uses bands of one row, as the reference):
 *   DSA_SCHED_ROW_BY_ROW             fetches = nnz
 *   DSA_SCHED_ROW_PARALLEL           per step t, one fetch per distinct t-th
 *                                    kept column of the band
 *   DSA_SCHED_ROW_PARALLEL_REORDERED one fetch per distinct column of the
 *                                    band (the column union)
 * and pe_idle_steps (sum of band max kept - own kept).  fetches / idle:
 * HOST arrays of cfg's pairs (per (b,h) pair).  The cost model SURVEY
 * 8(f) item 4 names for grouping query rows (bench reports the reordered
 * reuse nnz / fetches). */
typedef enum dsa_schedule {
    DSA_SCHED_ROW_BY_ROW = 0,
    DSA_SCHED_ROW_PARALLEL = 1,
    DSA_SCHED_ROW_PARALLEL_REORDERED = 2
} dsa_schedule;
dsa_status dsa_dataflow_trace(const dsa_config* cfg, const dsa_mask* mask, int32_t schedule, int64_t band,
                              uint64_t* fetches, uint64_t* idle, void* stream);

/* The reference's mask generators on a caller-held DENSE score matrix
 * (P/include/dsattn/maskgen.hpp:14-30), for callers that already hold S~:
 *   dsa_colvec_mask_f64     colvec_mask, column orientation (P/src/maskgen.cpp:
 *                           44-59): bands of v rows, band score of column j =
 *                           sum of |s(i, j)| over the band (rows in order),
 *                           row_topk_indices keeps `keep` columns per band;
 *                           band_cols is ceil(l / v) x keep (ascending).  NOTE
 *                           the reference rule here is SUM |s|; the BASELINE
 *                           C2 rule (max-pooled exact integer scores) is
 *                           DSA_MASK_COLVEC of dsa_select.
 *   dsa_threshold_mask_f64  threshold_mask (P/src/maskgen.cpp:22-31): keep[i][j]
 *                           = (value >= theta), value = s or its row softmax
 *                           (P/src/linalg.cpp:51-67; rounded to f32 when
 *                           round_f32); keep is rows x cols bytes.  The softmax
 *                           weights equal the reference's to the last ulp of
 *                           exp(), so a weight within an ulp of theta may differ.
 * scores: DEVICE f64 row-major; outputs DEVICE. */
dsa_status dsa_colvec_mask_f64(int64_t l, int64_t v, int64_t keep, const double* scores, uint32_t* band_cols,
                               void* stream);
dsa_status dsa_threshold_mask_f64(int64_t rows, int64_t cols, const double* scores, double theta,
                                  int32_t post_softmax, int32_t round_f32, uint8_t* keep, void* stream);

/* The reference's UNFUSED sparse operators, in its own value type (f64) and
 * CSR layout, for callers that use the three steps separately
 * (P/include/dsattn/sparse.hpp:47-55, P/src/sparse.cpp:38-91 over
 * P/src/kernels/scalar.cpp:34-58); the fused hot path is
 * dsa_sparse_attention.  All pointers are DEVICE pointers; rowptr has
 * rows + 1 entries (u64), cols the kept columns (u32, ascending per row).
 *   dsa_sddmm_f64           values[p] = <Q_i, K_cols[p]> (* 1/sqrt(d) when scale),
 *                           one fma per term in index order (the scalar kernel's
 *                           rounding: bit-identical to it)
 *   dsa_sparse_softmax_f64  max-subtracted softmax over each row's stored
 *                           entries, terms summed in entry order; an empty row
 *                           stays empty and is flagged in empty_rows (optional,
 *                           rows bytes, written 0 / 1)
 *   dsa_spmm_f64            Z_i = sum_p weights[p] V_cols[p] (fma in entry order),
 *                           empty rows give zero rows; z is rows x dv (f64)
 * Stream-ordered, no allocation, no host synchronisation. */
/* row_topk_indices on any f64 matrix (P/src/linalg.cpp:69-85; the reference's
 * oracle_topk_mask is this on the exact Q K^T, P/src/maskgen.cpp:11-16):
 * scores rows x cols (DEVICE, row-major), out rows x keep column indices
 * (DEVICE, ascending per row) -- value descending, the LOWEST column first
 * among equal values (-0 == +0), 1 <= keep <= cols <= 25600. */
dsa_status dsa_row_topk_f64(int64_t rows, int64_t cols, const double* scores, int64_t keep, uint32_t* out,
                            void* stream);
dsa_status dsa_sddmm_f64(int64_t rows, int64_t d, const double* q, const double* k, const uint64_t* rowptr,
                         const uint32_t* cols, int32_t scale, double* values, void* stream);
dsa_status dsa_sparse_softmax_f64(int64_t rows, const uint64_t* rowptr, const double* scores, double* weights,
                                  uint8_t* empty_rows, void* stream);
dsa_status dsa_spmm_f64(int64_t rows, int64_t dv, const uint64_t* rowptr, const uint32_t* cols, const double* weights,
                        const double* v, double* z, void* stream);

/* Exact operation counts for a computed mask (synchronises `stream`). */
dsa_status dsa_counters(const dsa_config* cfg, const dsa_mask* mask, dsa_counts* out,
                        void* stream);

/* ------------------------------------------------------ synthetic inputs */
/* Seeded BASELINE generator (host): Q/K/V ~ N(0,1), a shared unit vector u
 * added at +3 to `planted_per_mille`/1000 of the key positions and at +0.5 to
 * every query, optional local band (+1.0 score bias inside 32-row windows),
 * P ~ N(0, 1/k) rounded to f32.  Pair p is generated from its own substream,
 * so any pair range can be regenerated independently.  q/k/v receive
 * [npairs][L][d] in cfg->dtype; p (may be NULL) receives [d][k]. */
dsa_status dsa_generate(const dsa_config* cfg, uint64_t seed, int32_t planted_per_mille,
                        int32_t band_width, int64_t pair0, int64_t npairs, void* q, void* k,
                        void* v, float* p, int32_t threads);

#ifdef __cplusplus
}
#endif
#endif /* DSA_B200_H */
