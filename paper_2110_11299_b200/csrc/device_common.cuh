// Device-side helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dsa {

__device__ __forceinline__ double to_double(float x) { return static_cast<double>(x); }
__device__ __forceinline__ double to_double(__nv_bfloat16 x) {
    return static_cast<double>(__bfloat162float(x));
}
__device__ __forceinline__ float to_float(float x) { return x; }
__device__ __forceinline__ float to_float(__nv_bfloat16 x) { return __bfloat162float(x); }

template <class T>
__device__ __forceinline__ T from_float(float x);
template <>
__device__ __forceinline__ float from_float<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_float<__nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);
}

// Levels layout ("chunk-planar"): per (b,h) pair [KD/8][L][8] bf16, i.e.
// element (row r, column c) at ((c/8) * L + r) * 8 + c % 8.  A run of rows of
// one 8-column chunk is contiguous, so a 128-row tile of the K-major
// no-swizzle UMMA layout is KD/8 contiguous bulk copies.
__host__ __device__ __forceinline__ int64_t lvl_index(int64_t L, int64_t r, int c) {
    return ((static_cast<int64_t>(c >> 3) * L + r) << 3) + (c & 7);
}

// bf16 bits holding a small integer level -> int (exact for |v| <= 256).
__device__ __forceinline__ int level_to_int(uint16_t b) {
    return static_cast<int>(__uint_as_float(static_cast<uint32_t>(b) << 16));
}

// Reference round-half-away (P/src/kernels/scalar.cpp:11-17), operation for
// operation in double.
__device__ __forceinline__ double round_half_away(double x) {
    double t = trunc(x);
    double f = x - t;
    if (f >= 0.5) t += 1.0;
    if (f <= -0.5) t -= 1.0;
    return t;
}

// Orderable rank keys: SMALLER key = BETTER (kept first); ties are broken
// by the lower column index by every selection routine.
__device__ __forceinline__ uint32_t rank_key_i32(int32_t s) {
    return static_cast<uint32_t>(static_cast<int64_t>(INT32_MAX) - s);
}
__device__ __forceinline__ uint64_t rank_key_i64(int64_t s) {
    return static_cast<uint64_t>(INT64_MAX) - static_cast<uint64_t>(s);  // s >= -INT64_MAX
}
__device__ __forceinline__ uint64_t rank_key_f64(double v) {
    if (v == 0.0) v = 0.0;  // -0 == +0 under the reference comparator
    uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
    uint64_t o = (b >> 63) ? ~b : (b | (1ull << 63));  // ascending with v
    return ~o;
}

// Deterministic exp shared with the oracle (oracle/dsa_oracle.c
// dsa_oracle_exp): Cody-Waite reduction + degree-13 Horner, fma only.
__device__ __forceinline__ double det_exp(double x) {
    if (x < -50.0) return 0.0;
    if (x > 50.0) x = 50.0;
    const double log2e = 1.4426950408889634;
    const double ln2_hi = 6.93147180369123816490e-01;
    const double ln2_lo = 1.90821492927058770002e-10;
    double n = rint(x * log2e);
    double r = fma(-n, ln2_hi, x);
    r = fma(-n, ln2_lo, r);
    double p = 1.6059043836821613e-10;
    p = fma(p, r, 2.0876756987868100e-09);
    p = fma(p, r, 2.5052108385441720e-08);
    p = fma(p, r, 2.7557319223985888e-07);
    p = fma(p, r, 2.7557319223985893e-06);
    p = fma(p, r, 2.4801587301587302e-05);
    p = fma(p, r, 1.9841269841269841e-04);
    p = fma(p, r, 1.3888888888888889e-03);
    p = fma(p, r, 8.3333333333333332e-03);
    p = fma(p, r, 4.1666666666666664e-02);
    p = fma(p, r, 1.6666666666666666e-01);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    return scalbn(p, static_cast<int>(n));
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace dsa
