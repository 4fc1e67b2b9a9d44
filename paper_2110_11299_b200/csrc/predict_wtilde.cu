// Phase 1 on the reference's own predictor entry point (approx_scores /
// approx_scores_from_r, P/src/predictor.cpp:67-80):
//
//   R  = X P                         (once per sample, shared by the heads;
//                                     P/src/trainer.cpp:162)
//   Q~ = quantize(R W~_Q[h]),  K~ = quantize(R W~_K[h])   per head h
//
// Every product is the reference matmul's sequential fp64 FMA chain
// acc = fma(a[i][t], b[t][j], acc), t ascending from acc = 0
// (P/src/kernels/scalar.cpp:19-32), rounded through float when the
// operands are f32 Matrices (P/src/linalg.cpp:14-15, matrix.hpp:71-74), so
// the integer levels and per-tensor scales are bit-identical by
// construction.  Work is O(L k (d_model + 2 k)) fp64 FMAs per pair: tiny
// next to the score / selection phases, so one thread per output row.
#include "device_common.cuh"
#include "kernels.h"

namespace dsa {
namespace {

constexpr int kT = 128;

__device__ __forceinline__ double round_f32_if(double x, int f32) {
    return f32 ? static_cast<double>(static_cast<float>(x)) : x;
}

// R[b][i][:] = X[b][i][:] . P   (grid.x over batch * L rows)
template <int KD>
__global__ void __launch_bounds__(kT) r_kernel(const double* __restrict__ x, const double* __restrict__ p,
                                              int64_t rows, int64_t dm, int f32, double* __restrict__ r) {
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (row >= rows) return;
    double acc[KD];
#pragma unroll
    for (int j = 0; j < KD; ++j) acc[j] = 0.0;
    const double* xr = x + row * dm;
    for (int64_t t = 0; t < dm; ++t) {
        const double a = __ldg(xr + t);
        const double* pr = p + t * KD;
#pragma unroll
        for (int j = 0; j < KD; ++j) acc[j] = fma(a, __ldg(pr + j), acc[j]);
    }
#pragma unroll
    for (int j = 0; j < KD; ++j) r[row * KD + j] = round_f32_if(acc[j], f32);
}

// x = R W~ for one (pair = b * heads + h, Q|K) row; per-tensor scope
// stores x in the f64 scratch [pair][2][L][KD] and merges |x| into the
// tensor's amax (atomic max on the IEEE bits); per-row scope quantises the
// row in place.  grid = (ceil(L / kT), pairs, 2).
template <int KD>
__global__ void __launch_bounds__(kT)
    wtilde_kernel(const double* __restrict__ r, const double* __restrict__ wq, const double* __restrict__ wk,
                  int64_t heads, int64_t L, int f32, int per_row, double qmax, double* __restrict__ xout,
                  unsigned long long* __restrict__ amax, uint16_t* __restrict__ lq, uint16_t* __restrict__ lk,
                  double* __restrict__ sq, double* __restrict__ sk) {
    __shared__ double sw[KD * KD];
    const int which = blockIdx.z;
    const int64_t pair = blockIdx.y, b = pair / heads, h = pair % heads;
    const double* w = (which ? wk : wq) + h * KD * KD;
    for (int i = threadIdx.x; i < KD * KD; i += kT) sw[i] = w[i];
    __syncthreads();
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    double local = 0.0;
    if (row < L) {
        double acc[KD];
#pragma unroll
        for (int j = 0; j < KD; ++j) acc[j] = 0.0;
        const double* rr = r + (b * L + row) * KD;
#pragma unroll
        for (int t = 0; t < KD; ++t) {
            const double a = rr[t];
#pragma unroll
            for (int j = 0; j < KD; ++j) acc[j] = fma(a, sw[t * KD + j], acc[j]);
        }
#pragma unroll
        for (int j = 0; j < KD; ++j) {
            acc[j] = round_f32_if(acc[j], f32);
            local = fmax(local, fabs(acc[j]));
        }
        if (per_row) {
            const double s = local / qmax;
            uint16_t* o = (which ? lk : lq) + pair * L * KD;
#pragma unroll
            for (int j = 0; j < KD; ++j) {
                double v = 0.0;
                if (local != 0.0) v = fmin(fmax(round_half_away(acc[j] / s), -qmax), qmax);
                o[lvl_index(L, row, j)] = __bfloat16_as_ushort(__float2bfloat16_rn(static_cast<float>(v)));
            }
            (which ? sk : sq)[pair * L + row] = local == 0.0 ? 0.0 : s;
        } else {
            double* o = xout + ((pair * 2 + which) * L + row) * KD;
#pragma unroll
            for (int j = 0; j < KD; ++j) o[j] = acc[j];
        }
    }
    if (per_row) return;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) local = fmax(local, __shfl_xor_sync(0xffffffffu, local, off));
    if ((threadIdx.x & 31) == 0)
        atomicMax(amax + pair * 2 + which, static_cast<unsigned long long>(__double_as_longlong(local)));
}

template <int KD>
void launch(const WtildeArgs& a, cudaStream_t st) {
    if (a.x != nullptr) {
        const int64_t rows = a.batch * a.L;
        r_kernel<KD><<<static_cast<unsigned>(ceil_div_i(rows, kT)), kT, 0, st>>>(a.x, a.p, rows, a.dm, a.round_f32,
                                                                               a.r);
        note_launch();
    }
    const int64_t pairs = a.batch * a.heads;
    if (!a.per_row) cudaMemsetAsync(a.amax, 0, sizeof(unsigned long long) * 2 * pairs, st);
    const dim3 grid(static_cast<unsigned>(ceil_div_i(a.L, kT)), static_cast<unsigned>(pairs), 2);
    wtilde_kernel<KD><<<grid, kT, 0, st>>>(a.r, a.wq, a.wk, a.heads, a.L, a.round_f32, a.per_row, a.qmax, a.x64,
                                           a.amax, a.lq, a.lk, a.sq, a.sk);
    note_launch();
    if (!a.per_row) launch_quantize_x64(a.x64, a.amax, pairs, a.L, KD, a.qmax, a.lq, a.lk, a.sq, a.sk, st);
}

}  // namespace

void run_predict_wtilde(const WtildeArgs& a, cudaStream_t st) {
    switch (a.KD) {
        case 16: launch<16>(a, st); break;
        case 32: launch<32>(a, st); break;
        default: throw_unsupported("projection width k must be 16 or 32");
    }
}

}  // namespace dsa
