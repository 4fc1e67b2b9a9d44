// Phase 1: low-rank projection Q.P / K.P and symmetric quantisation.
//
// Bit-exactness contract: the integer levels must equal the
// reference's, whose projected value is the double sequential-FMA chain
// acc = fma(x[t], p[t][j], acc), t ascending (P/src/kernels/scalar.cpp:19-32),
// optionally rounded through float (P/src/linalg.cpp:15).  This kernel
// evaluates exactly that chain in fp64 (DFMA, same order), so every level --
// and the per-tensor amax / scale -- is bit-identical by construction.
//
// Layout: X = [pairs][L][D] (bf16 or f32), P = [D][KD] f32 (staged in smem as
// f64), levels = [pairs][L][KD] bf16 (exact small integers), scales f64.
#include <cuda_bf16.h>

#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"

namespace dsa {
namespace {

constexpr int kRowsPerCta = 128;

template <class T, int D, int KD>
__device__ __forceinline__ void project_row(const T* __restrict__ xrow, const double* sp,
                                            int round_f32, double (&acc)[KD]) {
#pragma unroll
    for (int j = 0; j < KD; ++j) acc[j] = 0.0;
    constexpr int kVec = 16 / sizeof(T);  // elements per 16-byte load
    const uint4* src = reinterpret_cast<const uint4*>(xrow);
#pragma unroll 1
    for (int t0 = 0; t0 < D; t0 += kVec) {
        uint4 raw = __ldg(src + t0 / kVec);
        const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int u = 0; u < kVec; ++u) {
            const double xv = to_double(e[u]);
            const double* prow = sp + (t0 + u) * KD;
#pragma unroll
            for (int j = 0; j < KD; ++j) acc[j] = fma(xv, prow[j], acc[j]);
        }
    }
    if (round_f32) {
#pragma unroll
        for (int j = 0; j < KD; ++j) acc[j] = static_cast<double>(static_cast<float>(acc[j]));
    }
}

template <int D, int KD>
__device__ __forceinline__ void stage_p(const float* __restrict__ p, double* sp) {
    for (int i = threadIdx.x; i < D * KD; i += blockDim.x) sp[i] = static_cast<double>(p[i]);
    __syncthreads();
}

__device__ __forceinline__ uint16_t level_bits(double r) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(static_cast<float>(r)));
}

// Per-tensor pass A: projected values to the f64 workspace + amax per
// (pair, Q|K) via an atomic max on the IEEE bits (non-negative doubles
// order like unsigned integers).  grid = (ceil(L/128), pairs, 2).
template <class T, int D, int KD>
__global__ void __launch_bounds__(kRowsPerCta)
    project_tensor_kernel(const T* __restrict__ q, const T* __restrict__ k,
                          const float* __restrict__ p, int64_t L, int round_f32,
                          double* __restrict__ xout, unsigned long long* __restrict__ amax) {
    __shared__ double sp[D * KD];
    stage_p<D, KD>(p, sp);
    const int which = blockIdx.z;
    const int64_t pair = blockIdx.y;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRowsPerCta + threadIdx.x;
    double local = 0.0;
    if (row < L) {
        const T* x = (which ? k : q) + (pair * L + row) * D;
        double acc[KD];
        project_row<T, D, KD>(x, sp, round_f32, acc);
        double* o = xout + ((pair * 2 + which) * L + row) * KD;
#pragma unroll
        for (int j = 0; j < KD; ++j) {
            o[j] = acc[j];
            local = fmax(local, fabs(acc[j]));
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
        local = fmax(local, __shfl_xor_sync(0xffffffffu, local, off));
    if ((threadIdx.x & 31) == 0)
        atomicMax(amax + pair * 2 + which, static_cast<unsigned long long>(__double_as_longlong(local)));
}

// Per-tensor pass B: s = amax / qmax, level = clamp(round_half_away(x / s))
// (P/src/predictor.cpp:37-43, P/src/kernels/scalar.cpp:60-68).
__global__ void quantize_tensor_kernel(const double* __restrict__ x,
                                       const unsigned long long* __restrict__ amax, int64_t L,
                                       int64_t KD, double qmax, uint16_t* __restrict__ lq,
                                       uint16_t* __restrict__ lk, double* __restrict__ sq,
                                       double* __restrict__ sk) {
    const int which = blockIdx.z;
    const int64_t pair = blockIdx.y;
    const double am = __longlong_as_double(static_cast<long long>(amax[pair * 2 + which]));
    const double s = am / qmax;
    if (blockIdx.x == 0 && threadIdx.x == 0) (which ? sk : sq)[pair] = am == 0.0 ? 0.0 : s;
    const int64_t n = L * KD;
    const double* xs = x + (pair * 2 + which) * n;
    uint16_t* out = (which ? lk : lq) + pair * n;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double r = 0.0;
        if (am != 0.0) {
            r = round_half_away(xs[i] / s);
            r = fmin(fmax(r, -qmax), qmax);
        }
        out[lvl_index(L, i / KD, static_cast<int>(i % KD))] = level_bits(r);
    }
}

// Per-row quantisation: one pass, scale per row.
template <class T, int D, int KD>
__global__ void __launch_bounds__(kRowsPerCta)
    project_rows_kernel(const T* __restrict__ q, const T* __restrict__ k,
                        const float* __restrict__ p, int64_t L, int round_f32, double qmax,
                        uint16_t* __restrict__ lq, uint16_t* __restrict__ lk,
                        double* __restrict__ sq, double* __restrict__ sk) {
    __shared__ double sp[D * KD];
    stage_p<D, KD>(p, sp);
    const int which = blockIdx.z;
    const int64_t pair = blockIdx.y;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRowsPerCta + threadIdx.x;
    if (row >= L) return;
    const T* x = (which ? k : q) + (pair * L + row) * D;
    double acc[KD];
    project_row<T, D, KD>(x, sp, round_f32, acc);
    double am = 0.0;
#pragma unroll
    for (int j = 0; j < KD; ++j) am = fmax(am, fabs(acc[j]));
    const double s = am / qmax;
    uint16_t* o = (which ? lk : lq) + pair * L * KD;
#pragma unroll
    for (int j = 0; j < KD; ++j) {
        double r = 0.0;
        if (am != 0.0) r = fmin(fmax(round_half_away(acc[j] / s), -qmax), qmax);
        o[lvl_index(L, row, j)] = level_bits(r);
    }
    (which ? sk : sq)[pair * L + row] = am == 0.0 ? 0.0 : s;
}

template <class T, int D, int KD>
void launch_predict(const PredictArgs& a, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>(ceil_div_i(a.L, kRowsPerCta)), static_cast<unsigned>(a.pairs), 2);
    const T* q = static_cast<const T*>(a.q);
    const T* k = static_cast<const T*>(a.k);
    if (a.per_row) {
        project_rows_kernel<T, D, KD><<<grid, kRowsPerCta, 0, st>>>(
            q, k, a.p, a.L, a.round_f32, a.qmax, a.lq, a.lk, a.sq, a.sk);
        note_launch();
    } else {
        cudaMemsetAsync(a.amax, 0, sizeof(unsigned long long) * 2 * a.pairs, st);
        project_tensor_kernel<T, D, KD><<<grid, kRowsPerCta, 0, st>>>(q, k, a.p, a.L, a.round_f32,
                                                                     a.xws, a.amax);
        const int64_t n = a.L * KD;
        const dim3 g2(static_cast<unsigned>(std::min<int64_t>(ceil_div_i(n, 256), 64)),
                      static_cast<unsigned>(a.pairs), 2);
        quantize_tensor_kernel<<<g2, 256, 0, st>>>(a.xws, a.amax, a.L, KD, a.qmax, a.lq, a.lk,
                                                   a.sq, a.sk);
        note_launch(2);
    }
}

template <class T, int D>
void dispatch_k(const PredictArgs& a, cudaStream_t st) {
    switch (a.KD) {
        case 16: launch_predict<T, D, 16>(a, st); break;
        case 32: launch_predict<T, D, 32>(a, st); break;
        default: throw_unsupported("projection width k must be 16 or 32");
    }
}

template <class T>
void dispatch_d(const PredictArgs& a, cudaStream_t st) {
    switch (a.D) {
        case 16: dispatch_k<T, 16>(a, st); break;
        case 32: dispatch_k<T, 32>(a, st); break;
        case 64: dispatch_k<T, 64>(a, st); break;
        case 128: dispatch_k<T, 128>(a, st); break;
        default: throw_unsupported("head dim d must be one of 16, 32, 64, 128");
    }
}

}  // namespace

void launch_quantize_x64(const double* x64, const unsigned long long* amax, int64_t pairs, int64_t L, int64_t KD,
                         double qmax, uint16_t* lq, uint16_t* lk, double* sq, double* sk, cudaStream_t st) {
    const dim3 g2(static_cast<unsigned>(std::min<int64_t>(ceil_div_i(L * KD, 256), 64)), static_cast<unsigned>(pairs), 2);
    quantize_tensor_kernel<<<g2, 256, 0, st>>>(x64, amax, L, KD, qmax, lq, lk, sq, sk);
    note_launch();
}

void run_predict(const PredictArgs& a, cudaStream_t st) {
    const bool force_dfma = options().predict_dfma;
    if (!force_dfma && predict_tensor_supported(a)) {
        run_predict_tensor(a, st);
        return;
    }
    if (!force_dfma && predict_tensor2_supported(a)) {
        run_predict_tensor2(a, st);
        return;
    }
    if (!force_dfma && predict_tc_supported(a)) {
        run_predict_tc(a, st);
        return;
    }
    if (!force_dfma && predict_fast_supported(a)) {
        run_predict_fast(a, st);
        return;
    }
    if (a.bf16) dispatch_d<__nv_bfloat16>(a, st);
    else dispatch_d<float>(a, st);
}

}  // namespace dsa
