// The reference's UNFUSED sparse operators on the device, in the reference's
// own f64 value type and CSR layout (P/src/sparse.cpp:38-91 over
// P/src/kernels/scalar.cpp:34-58): sddmm (scores at kept positions),
// sparse_softmax (max-subtracted row softmax over the stored entries, empty
// rows flagged), spmm (Z_i = sum_j a_ij V_j, empty rows zero).  They exist
// for callers that use the three operators separately (the fused hot path is
// dsa_sparse_attention); every accumulation follows the reference's scalar
// order with one fused multiply-add per term, so sddmm and spmm reproduce the
// reference's scalar kernels bit for bit and sparse_softmax to the last ulp
// of exp().
#include <cstdint>

#include "kernels.h"

namespace dsa {
namespace {

constexpr int kT = 256;

// one lane per kept position: acc = fma(q[t], k[t], acc) for t = 0..d-1, * scale
__global__ void __launch_bounds__(kT) sddmm_f64_kernel(const double* __restrict__ q, const double* __restrict__ k,
                                                       const uint64_t* __restrict__ rowptr,
                                                       const uint32_t* __restrict__ cols, int64_t rows, int64_t d,
                                                       double scale, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x) >> 5;
    if (row >= rows) return;
    const double* qr = q + row * d;
    const uint64_t b = rowptr[row], e = rowptr[row + 1];
    for (uint64_t p = b + lane; p < e; p += 32) {
        const double* kr = k + static_cast<int64_t>(cols[p]) * d;
        double acc = 0.0;
        for (int64_t t = 0; t < d; ++t) acc = fma(qr[t], kr[t], acc);
        out[p] = acc * scale;
    }
}

// one warp per row: max, exp(s - max), sum in entry order (lane partials are
// NOT used for the sum: the reference adds the terms sequentially)
__global__ void __launch_bounds__(kT) sparse_softmax_f64_kernel(const double* __restrict__ s,
                                                                const uint64_t* __restrict__ rowptr, int64_t rows,
                                                                double* __restrict__ w,
                                                                uint8_t* __restrict__ empty_rows) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x) >> 5;
    if (row >= rows) return;
    const uint64_t b = rowptr[row], e = rowptr[row + 1];
    if (b == e) {
        if (lane == 0 && empty_rows) empty_rows[row] = 1;
        return;
    }
    if (lane == 0 && empty_rows) empty_rows[row] = 0;
    double m = -INFINITY;
    for (uint64_t p = b + lane; p < e; p += 32) m = fmax(m, s[p]);
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    for (uint64_t p = b + lane; p < e; p += 32) w[p] = exp(s[p] - m);
    __syncwarp();
    // sequential sum in entry order (the reference's rounding): 32 entries per
    // step, lane l holds entry p0 + l, lane 0 folds them in order
    double sum = 0.0;
    for (uint64_t p0 = b; p0 < e; p0 += 32) {
        const uint64_t p = p0 + lane;
        const double x = p < e ? w[p] : 0.0;
        const int n = e - p0 < 32 ? static_cast<int>(e - p0) : 32;
        for (int i = 0; i < n; ++i) sum += __shfl_sync(0xffffffffu, x, i);
    }
    for (uint64_t p = b + lane; p < e; p += 32) w[p] = w[p] / sum;
}

// one thread per output element (row, column): z = fma(w_p, V[col_p][c], z) in entry order
__global__ void __launch_bounds__(kT) spmm_f64_kernel(const double* __restrict__ w,
                                                      const uint64_t* __restrict__ rowptr,
                                                      const uint32_t* __restrict__ cols, int64_t rows,
                                                      const double* __restrict__ v, int64_t dv,
                                                      double* __restrict__ z) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (idx >= rows * dv) return;
    const int64_t row = idx / dv, c = idx - row * dv;
    double acc = 0.0;
    for (uint64_t p = rowptr[row]; p < rowptr[row + 1]; ++p)
        acc = fma(w[p], v[static_cast<int64_t>(cols[p]) * dv + c], acc);
    z[idx] = acc;
}

// colvec_mask's band scores on a caller-held S~ (P/src/maskgen.cpp:52-58):
// pooled[band][j] = sum over the band's rows of |s(i, j)|, rows added in
// order (the reference's rounding).  One thread per (band, column).
__global__ void __launch_bounds__(kT) band_abs_sum_f64_kernel(const double* __restrict__ s, int64_t l, int64_t v,
                                                              int64_t nb, double* __restrict__ pooled) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (idx >= nb * l) return;
    const int64_t band = idx / l, j = idx - band * l;
    const int64_t r1 = min((band + 1) * v, l);
    double acc = 0.0;
    for (int64_t i = band * v; i < r1; ++i) acc += fabs(s[i * l + j]);
    pooled[idx] = acc;
}

// threshold_mask on a caller-held matrix (P/src/maskgen.cpp:22-31): keep[i][j]
// = value >= theta, the value being s itself or its row softmax
// (P/src/linalg.cpp:51-67: max-subtracted exp, terms summed in column order,
// rounded to f32 when the matrix is).  One warp per row.
__global__ void __launch_bounds__(kT) threshold_f64_kernel(const double* __restrict__ s, int64_t rows, int64_t cols,
                                                           double theta, int post_softmax, int f32,
                                                           double* __restrict__ scratch, uint8_t* __restrict__ keep) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x) >> 5;
    if (row >= rows) return;
    const double* r = s + row * cols;
    uint8_t* k = keep + row * cols;
    if (!post_softmax) {
        for (int64_t j = lane; j < cols; j += 32) k[j] = r[j] >= theta;
        return;
    }
    double* e = scratch + row * cols;
    double m = -INFINITY;
    for (int64_t j = lane; j < cols; j += 32) m = fmax(m, r[j]);
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    for (int64_t j = lane; j < cols; j += 32) e[j] = exp(r[j] - m);
    __syncwarp();
    double sum = 0.0;
    for (int64_t j0 = 0; j0 < cols; j0 += 32) {
        const double x = j0 + lane < cols ? e[j0 + lane] : 0.0;
        const int n = cols - j0 < 32 ? static_cast<int>(cols - j0) : 32;
        for (int i = 0; i < n; ++i) sum += __shfl_sync(0xffffffffu, x, i);
    }
    for (int64_t j = lane; j < cols; j += 32) {
        double p = e[j] / sum;
        if (f32) p = static_cast<double>(static_cast<float>(p));
        k[j] = p >= theta;
    }
}

unsigned blocks_for(int64_t threads) { return static_cast<unsigned>((threads + kT - 1) / kT); }

}  // namespace

void run_sddmm_f64(const double* q, const double* k, const uint64_t* rowptr, const uint32_t* cols, int64_t rows,
                   int64_t d, double scale, double* out, cudaStream_t st) {
    if (rows == 0) return;
    sddmm_f64_kernel<<<blocks_for(rows * 32), kT, 0, st>>>(q, k, rowptr, cols, rows, d, scale, out);
    note_launch(1);
}

void run_sparse_softmax_f64(const double* s, const uint64_t* rowptr, int64_t rows, double* w, uint8_t* empty_rows,
                            cudaStream_t st) {
    if (rows == 0) return;
    sparse_softmax_f64_kernel<<<blocks_for(rows * 32), kT, 0, st>>>(s, rowptr, rows, w, empty_rows);
    note_launch(1);
}

void run_spmm_f64(const double* w, const uint64_t* rowptr, const uint32_t* cols, int64_t rows, const double* v,
                  int64_t dv, double* z, cudaStream_t st) {
    if (rows == 0 || dv == 0) return;
    spmm_f64_kernel<<<blocks_for(rows * dv), kT, 0, st>>>(w, rowptr, cols, rows, v, dv, z);
    note_launch(1);
}

void run_band_abs_sum_f64(const double* s, int64_t l, int64_t v, double* pooled, cudaStream_t st) {
    const int64_t nb = (l + v - 1) / v;
    band_abs_sum_f64_kernel<<<blocks_for(nb * l), kT, 0, st>>>(s, l, v, nb, pooled);
    note_launch(1);
}

void run_threshold_f64(const double* s, int64_t rows, int64_t cols, double theta, int post_softmax, int f32,
                       double* scratch, uint8_t* keep, cudaStream_t st) {
    threshold_f64_kernel<<<blocks_for(rows * 32), kT, 0, st>>>(s, rows, cols, theta, post_softmax, f32, scratch, keep);
    note_launch(1);
}

}  // namespace dsa
