// Host-visible launch interfaces of the device kernels (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

namespace dsa {

[[noreturn]] void throw_unsupported(const std::string& what);
[[noreturn]] void throw_cuda(cudaError_t e, const char* where);
// Counts kernel launches of this library (dsa_launch_counter()).
void note_launch(int n = 1);
// Multiprocessor count of the current device (cached per device).
int sm_count();

// Kernel-selection switches, read from the environment ONCE when the
// library loads (never per call).  Each forces a slower, simpler kernel so
// the parity tests can cover it; the defaults are the measured-fastest path.
struct Options {
    bool attn_generic;       // DSA_ATTN_GENERIC: attn_rows_generic for every mask
    bool threshold_generic;  // DSA_THRESHOLD_GENERIC: CTA-per-row threshold kernels
    bool block_generic;      // DSA_BLOCK_GENERIC: CTA-per-row block selection
    bool topk_generic;       // DSA_TOPK_GENERIC: CTA-per-row radix top-k
    bool predict_dfma;       // DSA_PREDICT_DFMA: exact fp64 projection chain
    bool fuse;               // DSA_FUSE: COLVEC select + attention in one kernel (measured slower on C2)
    bool block_tc;           // DSA_BLOCK_TC: tcgen05 + TMA block attention (measured slower on C3)
    bool predict_tiles;      // DSA_PREDICT_TILES: tile kernels instead of the one-CTA-per-tensor pass
    bool block_cpasync;      // DSA_BLOCK_CPASYNC: block attention with cp.async staging instead of TMA
    int pipeline_chunks;     // DSA_PIPELINE_CHUNKS: pair chunks overlapped on 3 streams
};
const Options& options();

inline int64_t ceil_div_i(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct PredictArgs {
    const void* q;
    const void* k;
    const float* p;
    int64_t pairs, L, D, KD;
    int bf16, per_row, round_f32;
    double qmax;
    uint16_t* lq;
    uint16_t* lk;
    double* sq;
    double* sk;
    double* xws;                // per-tensor: [pairs][2][L][KD] f64 scratch
    unsigned long long* amax;  // per-tensor: [pairs][2]
    unsigned char* pimg;       // tensor-core path: P-split operand image
    float* xhat;               // tensor-core path: x^ [pairs][2][L][KD] + bound factors [pairs][2][L]
};
// x^ scratch per pair (floats): x^ [2][L][KD] + bound factors [2][L] + a
// share of the deferred-recompute list (u64 entries, 1/8 of the levels)
// and of its counter.  Layout of a call's view over n pairs: x^ of all n,
// factors of all n, the counter (u64), then the list (capacity n L KD / 4).
// Rounded up to 64 floats (256 B) so a chunk's view at any pair0 keeps the
// float4 / u64 alignment of its parts.
inline int64_t xhat_floats_per_pair(int64_t L, int64_t KD) {
    return (2 * L * (KD + 1) + L * KD / 2 + 2 + 63) / 64 * 64;
}
void run_predict(const PredictArgs& a, cudaStream_t st);
bool predict_fast_supported(const PredictArgs& a);
void run_predict_fast(const PredictArgs& a, cudaStream_t st);
bool predict_tc_supported(const PredictArgs& a);
size_t predict_tc_image_bytes(int64_t D, int64_t KD);
void run_predict_tc(const PredictArgs& a, cudaStream_t st);
bool predict_tensor_supported(const PredictArgs& a);
void run_predict_tensor(const PredictArgs& a, cudaStream_t st);
bool predict_tensor2_supported(const PredictArgs& a);
void run_predict_tensor2(const PredictArgs& a, cudaStream_t st);

// approx_scores_from_r with the per-head k x k W~ (P/src/predictor.cpp:67-80)
struct WtildeArgs {
    int64_t batch, heads, L, dm, KD;
    const double* x;   // [batch][L][dm] or null (r is then the input)
    const double* p;   // [dm][KD]
    double* r;         // [batch][L][KD]
    const double* wq;  // [heads][KD][KD]
    const double* wk;
    int round_f32, per_row;
    double qmax;
    uint16_t* lq;
    uint16_t* lk;
    double* sq;
    double* sk;
    double* x64;                // per-tensor scratch [pairs][2][L][KD]
    unsigned long long* amax;   // [pairs][2]
};
void run_predict_wtilde(const WtildeArgs& a, cudaStream_t st);
// per-tensor pass B over an f64 projection scratch [pairs][2][L][KD]
void launch_quantize_x64(const double* x64, const unsigned long long* amax, int64_t pairs, int64_t L, int64_t KD,
                         double qmax, uint16_t* lq, uint16_t* lk, double* sq, double* sk, cudaStream_t st);

enum SelectMode { kRowTopk = 0, kColvec = 1, kBlock = 2, kThreshold = 3 };

struct SelectArgs {
    int mode;
    int64_t pairs, L, KD, D;
    int per_row;
    const uint16_t* lq;
    const uint16_t* lk;
    const double* sq;
    const double* sk;
    int64_t keep;
    int64_t vec_v;
    int64_t block;
    int force_diag;
    int causal;
    int64_t frac_num, frac_den, cap;
    int qmax;
    uint32_t* cols;
    uint64_t* rowptr;   // threshold: [pairs*L + 1]
    int64_t capacity;
    uint8_t* empty_rows;
    // scratch
    int32_t* pooled;    // block: [pairs][2][nb][KD]
    int64_t* etab;      // threshold: [pairs][span]
    uint64_t* counts;   // threshold: [pairs*L]
    int2* cut;          // threshold: [pairs*L] {v_cut, tie quota}
    unsigned* ovf_n;    // per-row top-k: overflow row count
    int64_t* ovf_list;  // per-row top-k: overflow rows [pairs*L]
    int64_t span;
    void* scan_tmp;
    size_t scan_tmp_bytes;
};
void run_select(const SelectArgs& a, cudaStream_t st);
size_t select_scan_tmp_bytes(int64_t n);
bool colvec_tc_supported(const SelectArgs& a);
void run_colvec_tc(const SelectArgs& a, cudaStream_t st);
bool threshold_tc_supported(const SelectArgs& a);
bool topk_rowsel_supported(const SelectArgs& a);
void run_topk_rowsel(const SelectArgs& a, cudaStream_t st);
void launch_topk_scaled_list(const SelectArgs& a, const int64_t* list, const unsigned* nlist, cudaStream_t st);
void run_threshold_tc(const SelectArgs& a, cudaStream_t st);
void launch_exp_table(const SelectArgs& a, cudaStream_t st);
void scan_counts(const SelectArgs& a, cudaStream_t st);

// fused per-head Q/K/V (+ predictor input) projection GEMM
struct QkvGemmArgs {
    int64_t batch, L, d_model, heads, dk, dv, npred;
    const void* x;   // [batch][L][d_model] bf16
    const void* w;   // [heads*(2 dk + dv) + npred][d_model] bf16
    void* q;         // [batch*heads][L][dk] bf16
    void* k;
    void* v;         // [batch*heads][L][dv] bf16
    float* r;        // [batch][L][npred] f32 (may be null when npred == 0)
};
void run_qkv_gemm(const QkvGemmArgs& g, cudaStream_t st);

struct AttnArgs {
    int mode;
    int64_t pairs, L, D;
    int bf16, scale;
    const void* q;
    const void* k;
    const void* v;
    const uint32_t* cols;
    const uint64_t* rowptr;
    int64_t keep, vec_v, block;
    void* z;
    uint8_t* empty_rows;
};
void run_attention(const AttnArgs& a, cudaStream_t st);
// prediction_accuracy counts {intersection, total, rows with unequal counts}
void run_prediction_accuracy(const AttnArgs& pred, const AttnArgs& orc, unsigned long long* out, cudaStream_t st);
void run_dataflow(const AttnArgs& m, int band, int kind, unsigned long long* fetches, unsigned long long* idle,
                  cudaStream_t st);
// row_topk_indices on an f64 matrix (select.cu)
void run_row_topk_f64(const double* s, int64_t rows, int64_t cols, int64_t keep, uint32_t* out, cudaStream_t st);
// the reference's unfused f64 operators on CSR (sparse_ops.cu)
void run_sddmm_f64(const double* q, const double* k, const uint64_t* rowptr, const uint32_t* cols, int64_t rows,
                   int64_t d, double scale, double* out, cudaStream_t st);
void run_sparse_softmax_f64(const double* s, const uint64_t* rowptr, int64_t rows, double* w, uint8_t* empty_rows,
                            cudaStream_t st);
void run_spmm_f64(const double* w, const uint64_t* rowptr, const uint32_t* cols, int64_t rows, const double* v,
                  int64_t dv, double* z, cudaStream_t st);
void run_band_abs_sum_f64(const double* s, int64_t l, int64_t v, double* pooled, cudaStream_t st);
void run_threshold_f64(const double* s, int64_t rows, int64_t cols, double theta, int post_softmax, int f32,
                       double* scratch, uint8_t* keep, cudaStream_t st);
bool band_attention_supported(const AttnArgs& a);
// block masks, 32 x 32 blocks, d = 128: tcgen05 + TMA (attention_block_tc.cu)
bool block_tc_supported(const AttnArgs& a);
void run_block_tc(const AttnArgs& a, cudaStream_t st);
void run_band_attention(const AttnArgs& a, cudaStream_t st);
// fused COLVEC select + band attention (mask optional): dsa_pipeline
bool colvec_fused_supported(const SelectArgs& s, const AttnArgs& a);
void run_colvec_fused(const SelectArgs& s, const AttnArgs& a, cudaStream_t st);

}  // namespace dsa
