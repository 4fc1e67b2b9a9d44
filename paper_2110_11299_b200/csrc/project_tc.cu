// Phase 1 on the 5th-gen tensor cores: projection + quantisation with levels
// certified bit-identical to the reference's (bf16 inputs).
//
// The reference level is clamp(round_half_away(x64 / s)), x64 the double
// sequential-FMA chain of the row against P (P/src/kernels/scalar.cpp:19-32)
// and s = max|x64| / qmax over the (b,h) tensor (P/src/predictor.cpp:37-43).
//
//   * P (f32) is split EXACTLY into three bf16 parts P = P1 + P2 + P3 (8 + 8 +
//     8 significant bits), so every product q * Pi is exact and
//       x^ = X . [P1 | P2 | P3]   (tcgen05.mma kind::f16, M = 128 rows,
//                                  N = 3 k, K = d, fp32 accumulation in TMEM)
//     is x up to fp32 accumulation rounding: |x^ - x64| <= e with
//       e = d 2^-22 |q| |p_j| + |x^| 2^-23 (+ one f32 ulp when the reference
//           rounds the product through float)  -- twice the worst-case
//     fp32 accumulation bound, so truncating adders are covered too;
//   * amax pass: per CTA, only elements with |x^| + e >= max(|x^| - e) can
//     hold the CTA's maximum; they are recomputed with the reference's own
//     fp64 chain and the exact maximum is merged per tensor with an atomic
//     max on its IEEE bits -- the global maximum's element is always a
//     candidate of its own CTA, so no second candidate pass is needed;
//   * quantise pass: t = x^ / s is certified when it is farther than the
//     scaled bound from every .5 rounding boundary, else the level is
//     recomputed exactly (a few in 10^4).
//
// One CTA = 128 rows of one tensor of one pair (thread = row = TMEM lane);
// X tiles arrive by 16-byte cp.async into the K-major no-swizzle layout, the
// P-split operand image (built once per call by psplit_kernel) by cp.async
// from L2, one MMA batch per CTA; many CTAs per SM overlap each other's
// loads.  Uncertified elements: in the two-read quantise pass (8-bit levels)
// and the per-row pass they go to a shared list recomputed by the whole CTA
// (the reference chain is sequential, so one element per thread); in the
// streaming x^ pass (<= 4-bit levels) they go to a global deferred list
// (one atomic per warp that has any) that quantize_fix_kernel recomputes, one thread per
// entry, grid = 2 x SM count.  When the list is full the streaming pass
// recomputes the level in place.
// HBM traffic: Q and K read twice (amax pass, quantise pass) or once plus
// the x^ round trip, levels written once.
#include <cuda_bf16.h>


#include "device_common.cuh"
#include "kernels.h"
#include "tc_sm100.cuh"

#ifndef DSA_ABLATE  // profiling builds only (tools/ablate.py); 0 in the library
#define DSA_ABLATE 0
#endif

namespace dsa {
namespace {

constexpr int kRows = 128;  // rows per CTA = threads = UMMA M

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0));
}

// K-major no-swizzle canonical layout of a [rows][D] bf16 operand: 8-row x
// 16-byte core matrices, K-adjacent cores 128 B apart (LBO), 8-row groups
// D * 16 B apart (SBO).
template <int D>
__device__ __forceinline__ uint32_t opnd_off(int r, int c) {
    return static_cast<uint32_t>((r >> 3) * (D * 16) + (c >> 3) * 128 + (r & 7) * 16 + (c & 7) * 2);
}

// the reference's fp64 chain (P read as f32 -> f64, exact), the row read
// from the staged operand tile
template <int D, int KD>
__device__ __forceinline__ double ref_chain_s(const unsigned char* xa, int r, const float* __restrict__ p, int j,
                                              int round_f32) {
    double acc = 0.0;
#pragma unroll 8
    for (int t = 0; t < D; ++t) {
        const __nv_bfloat16 xv = *reinterpret_cast<const __nv_bfloat16*>(xa + opnd_off<D>(r, t));
        acc = fma(to_double(xv), static_cast<double>(__ldg(p + t * KD + j)), acc);
    }
    return round_f32 ? static_cast<double>(static_cast<float>(acc)) : acc;
}

constexpr int kMaxList = 1024;  // uncertified (row, column) entries recomputed cooperatively

// Level of element (row r, column j) of the staged tile, bit-identical to
// the reference's clamp(round_half_away(chain / s)) (chain = the sequential
// fp64 fma chain of ref_chain_s) without walking that d-long dependent
// chain: the d products x_t p_tj are exact in fp64 (bf16 x f32: <= 32
// significant bits) and are summed into 8 independent partial sums, then
// combined pairwise.  That sum and the chain are both within (steps)
// 2^-53 sum|x_t p_tj| of the exact dot product, so |chain - sum| <=
// (d + d/8 + 3) 2^-53 sum|.| (widened by 1 %); when both ends of that
// interval, scaled by 1/s (plus 2^-50 relative for the reciprocal's and the
// reference division's rounding), round to the same level, it is the
// reference's.  Otherwise (a quotient within ~1e-14 relative of a .5
// boundary) the sequential chain itself.
template <int D, int KD>
__device__ __forceinline__ float level_split(const unsigned char* xa, int r, const float* __restrict__ p, int j,
                                             double s, double inv_s, double qmax) {
    double ps[8], pa[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) ps[u] = pa[u] = 0.0;
#pragma unroll
    for (int t0 = 0; t0 < D; t0 += 8) {
        const uint4 xv = *reinterpret_cast<const uint4*>(xa + opnd_off<D>(r, t0));  // 8 consecutive t
        const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(&xv);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double pr = to_double(xb[u]) * static_cast<double>(__ldg(p + (t0 + u) * KD + j));
            ps[u] += pr;
            pa[u] += fabs(pr);
        }
    }
#pragma unroll
    for (int w = 4; w >= 1; w >>= 1)
#pragma unroll
        for (int u = 0; u < w; ++u) {
            ps[u] += ps[u + w];
            pa[u] += pa[u + w];
        }
    const double sum = ps[0];
    const double e = pa[0] * (static_cast<double>(D + D / 8 + 3) * 1.1102230246251565e-16 * 1.01) + 1e-300;
    const double dq = fabs(sum * inv_s) * 8.881784197001252e-16;  // 2^-50 |q|
    const double lo = fmin(fmax(round_half_away((sum - e) * inv_s - dq), -qmax), qmax);
    const double hi = fmin(fmax(round_half_away((sum + e) * inv_s + dq), -qmax), qmax);
    if (lo == hi) return static_cast<float>(lo);
    // within the bound of a .5 boundary: the reference's own chain
    return static_cast<float>(fmin(fmax(round_half_away(ref_chain_s<D, KD>(xa, r, p, j, 0) / s), -qmax), qmax));
}

__device__ __forceinline__ float xbound(float x, float qp, int round_f32, float dscale) {
    return fmaf(qp, dscale, fabsf(x) * (round_f32 ? 2.4e-7f : 1.2e-7f)) + 1e-30f;
}

// Certified level, or NaN when t = x/s may round differently from the
// reference's (fp32 arithmetic; the margin covers the bound and the fp32
// rounding of x * (1/s)).  With e = dq p_j + |x| rel, the scaled margin
// e inv_s 1.001 + |t| 1e-6 is folded to  |t| K1 + B_j  where
// K1 = 1e-6 + 1.001 rel and B_j = 1.001 dq inv_s p_j (per row and column).
__device__ __forceinline__ float cert_level(float x, float bj, float k1, float inv_s, float qmax) {
    const float t = x * inv_s;
    const float at = fabsf(t);
    const float frac = at - floorf(at);
    const float margin = fmaf(at, k1, bj) + 1e-30f;
    if (fabsf(frac - 0.5f) <= margin) return __int_as_float(0x7fc00000);
    return fminf(fmaxf(copysignf(floorf(at + 0.5f), t), -qmax), qmax);
}

template <int D, int KD, int R = kRows, bool ROW = false>
struct ProjSmem {
    static constexpr int N = 3 * KD;                 // B rows: P1 | P2 | P3 columns
    static constexpr int kX = R * D * 2;             // X tile (R rows)
    static constexpr int kB = N * D * 2;             // P-split image
    static constexpr int kImg = kB + KD * 4;         // image + |p_j| (bound factors)
    static constexpr int kLvl = R * KD * 2;          // staged levels [row][KD] bf16
    static constexpr int kList = kMaxList * 4;
    static constexpr int kMisc = 64;
    static constexpr int kRowMax = ROW ? R * 8 : 0;  // per-row exact max (ROW scope)
    static constexpr int bytes() { return kX + kImg + kMisc + kLvl + kList + kRowMax; }
};

// P -> exact three-way bf16 split in the B-operand layout + |p_j| * 1.001
// (one CTA; the image is the same for every pair).
template <int D, int KD>
__global__ void psplit_kernel(const float* __restrict__ p, unsigned char* __restrict__ img,
                              unsigned long long* __restrict__ amax, int64_t namax,
                              unsigned long long* __restrict__ lcnt) {
    using Sm = ProjSmem<D, KD>;
    if (lcnt != nullptr && threadIdx.x == 0) *lcnt = 0ull;  // deferred-recompute list
    if (amax != nullptr)
        for (int64_t i = threadIdx.x; i < namax; i += blockDim.x) amax[i] = 0ull;  // amax pass accumulators
    __shared__ float p_s[D * KD];  // P staged once: the norm chains below read it from shared memory
    for (int i = threadIdx.x; i < D * KD; i += blockDim.x) {
        const int c = i / KD, j = i % KD;
        const float v = __ldg(p + i);
        p_s[i] = v;
        const __nv_bfloat16 b1 = __float2bfloat16_rn(v);
        const float r1 = v - __bfloat162float(b1);
        const __nv_bfloat16 b2 = __float2bfloat16_rn(r1);
        const float r2 = r1 - __bfloat162float(b2);
        const __nv_bfloat16 b3 = __float2bfloat16_rn(r2);
        *reinterpret_cast<__nv_bfloat16*>(img + opnd_off<D>(j, c)) = b1;
        *reinterpret_cast<__nv_bfloat16*>(img + opnd_off<D>(KD + j, c)) = b2;
        *reinterpret_cast<__nv_bfloat16*>(img + opnd_off<D>(2 * KD + j, c)) = b3;
    }
    __syncthreads();
    if (threadIdx.x < KD) {
        double s2 = 0.0;
        for (int u = 0; u < D; ++u) {
            const double v = static_cast<double>(p_s[u * KD + threadIdx.x]);
            s2 = fma(v, v, s2);
        }
        reinterpret_cast<float*>(img + Sm::kB)[threadIdx.x] = static_cast<float>(sqrt(s2) * 1.001);
    }
}

// QUANT = false: exact per-tensor amax (atomic max into amax[pair][2]).
// QUANT = true : levels (chunk-planar) + scales from the exact amax.
// grid = (row tiles, 2 tensors, pairs)
// R = 128 or 256 rows per CTA (one or two M = 128 MMAs; two halves amortise
// the P-image copy and the CTA prologue over twice the rows).
// ROW = true: per-row scale (quant_scope = row) in ONE pass:
// the row's exact max from its candidates, then its levels and scale.
template <int D, int KD, bool QUANT, int R = kRows, bool ROW = false>
__global__ void __launch_bounds__(R)
    project_tc_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                      const float* __restrict__ p, const unsigned char* __restrict__ img, int64_t L,
                      int round_f32, double qmax, unsigned long long* __restrict__ amax,
                      uint16_t* __restrict__ lq, uint16_t* __restrict__ lk, double* __restrict__ sq,
                      double* __restrict__ sk, float* __restrict__ xhat) {
    using Sm = ProjSmem<D, KD, R, ROW>;
    constexpr int N = Sm::N;
    constexpr int TC = (R / 128) * N <= 64 ? 64 : ((R / 128) * N <= 128 ? 128 : 256);  // TMEM columns
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* xa = smem;
    unsigned char* pb = smem + Sm::kX;
    const float* pn = reinterpret_cast<const float*>(pb + Sm::kB);
    uint64_t* bar = reinterpret_cast<uint64_t*>(pb + Sm::kImg);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    unsigned int* red_f = tslot + 1;                                   // CTA max(|x| - e), float bits
    unsigned long long* red_d = reinterpret_cast<unsigned long long*>(bar + 3);  // CTA exact max
    unsigned int* lcount = reinterpret_cast<unsigned int*>(bar + 4);
    uint16_t* lvl_s = reinterpret_cast<uint16_t*>(pb + Sm::kImg + Sm::kMisc);
    uint32_t* list = reinterpret_cast<uint32_t*>(pb + Sm::kImg + Sm::kMisc + Sm::kLvl);
    unsigned long long* rowmax = reinterpret_cast<unsigned long long*>(pb + Sm::kImg + Sm::kMisc + Sm::kLvl + Sm::kList);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int which = blockIdx.y;
    const int64_t pair = blockIdx.z;
    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * R;
    const __nv_bfloat16* X = (which ? k : q) + pair * L * D;

    if (tid == 0) {
        tc::mbar_init(bar, 1);
        tc::fence_barrier_init();
        *red_f = 0u;
        *red_d = 0ull;
        *lcount = 0u;
    }
    if (warp == 0) tc::tmem_alloc<TC>(tslot);
    {
        // X tile: 16-byte chunks, 8 consecutive threads = 8 rows of one chunk
        constexpr int kCh = D / 8;
        const uint32_t xs = tc::smem_addr(xa);
        for (int i = tid; i < R * kCh; i += R) {
            const int r7 = i & 7, ch = (i >> 3) % kCh, rg = (i >> 3) / kCh;
            const int r = rg * 8 + r7;
            const bool ok = row0 + r < L;
            cp16(xs + opnd_off<D>(r, ch * 8), X + (ok ? row0 + r : 0) * D + ch * 8, ok);
        }
        // P-split image (+ |p_j|)
        const uint32_t ps = tc::smem_addr(pb);
        for (int i = tid; i < Sm::kImg / 16; i += R) cp16(ps + i * 16, img + i * 16, true);
        asm volatile("cp.async.commit_group;\n");
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tslot;
    if (tid == 0) {
        constexpr uint32_t idesc = tc::idesc_bf16_f32(128, N);
        const uint32_t xs = tc::smem_addr(xa), bs = tc::smem_addr(pb);
#pragma unroll
        for (int h = 0; h < R / 128; ++h)  // rows 128h.. -> TMEM columns [hN, hN + N)
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
                const uint64_t ad = tc::desc_kmajor_nosw(xs + h * 16 * (D * 16) + ks * 256, 128, D * 16);
                const uint64_t bd = tc::desc_kmajor_nosw(bs + ks * 256, 128, D * 16);
                tc::mma_bf16(tmem + h * N, ad, bd, idesc, ks > 0);
            }
        tc::commit(bar);
    }
    // |q| of this thread's row (bound factor), from the staged tile
    const int64_t r = row0 + tid;
    const bool valid = r < L;
    float nq;
    {
        float s2 = 0.f;
#pragma unroll
        for (int ch = 0; ch < D / 8; ++ch) {
            const uint4 v = *reinterpret_cast<const uint4*>(xa + opnd_off<D>(tid, ch * 8));
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float2 f = __bfloat1622float2(h[u]);
                s2 = fmaf(f.x, f.x, fmaf(f.y, f.y, s2));
            }
        }
        nq = sqrtf(s2) * 1.001f + 1e-30f;
    }
    const float dq = nq * (static_cast<float>(D) * 2.384185791015625e-7f);  // |q| d 2^-22
    const float rel = round_f32 ? 2.4e-7f : 1.2e-7f;
    tc::mbar_wait(bar, 0);
    tc::fence_after_sync();
    // x^_j = P1 part + (P2 part + P3 part)
    float xv[KD];
    {
        const uint32_t base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * N;
        uint32_t d0[32];
        if constexpr (N == 48) {
            uint32_t d1[16];
            tc::ld_32x32b_x32(base, d0);
            tc::ld_32x32b_x16(base + 32, d1);
            tc::wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j)
                xv[j] = __uint_as_float(d0[j]) + (__uint_as_float(d0[16 + j]) + __uint_as_float(d1[j]));
        } else {
            uint32_t d1[32], d2[32];
            tc::ld_32x32b_x32(base, d0);
            tc::ld_32x32b_x32(base + 32, d1);
            tc::ld_32x32b_x32(base + 64, d2);
            tc::wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j)
                xv[j] = __uint_as_float(d0[j]) + (__uint_as_float(d1[j]) + __uint_as_float(d2[j]));
        }
    }
    tc::fence_before_sync();
    if constexpr (ROW) {
        // row max candidates: |x^_j| + e_j >= max_j(|x^_j| - e_j), one bound
        // per row (e_j <= E_row); recomputed exactly by the whole CTA
        float xm = 0.f, pm = 0.f;
#pragma unroll
        for (int j = 0; j < KD; ++j) {
            xm = fmaxf(xm, fabsf(xv[j]));
            pm = fmaxf(pm, pn[j]);
        }
        const float er = fmaf(dq, pm, xm * rel) + 1e-30f;
        const float thr = fmaxf(0.f, (xm - er) * 0.999999f) - er;
        rowmax[tid] = 0ull;
#pragma unroll
        for (int j = 0; j < KD; ++j)
            if (valid && fabsf(xv[j]) >= thr) {
                const unsigned slot = atomicAdd(lcount, 1u);
                if (slot < kMaxList) list[slot] = (static_cast<uint32_t>(tid) << 6) | j;
                else atomicMax(&rowmax[tid], static_cast<unsigned long long>(__double_as_longlong(
                                                 fabs(ref_chain_s<D, KD>(xa, tid, p, j, round_f32)))));
            }
        __syncthreads();
        {
            const unsigned n = min(*lcount, static_cast<unsigned>(kMaxList));
            for (unsigned e = tid; e < n; e += R) {
                const int rr = static_cast<int>(list[e] >> 6);
                const double v = fabs(ref_chain_s<D, KD>(xa, rr, p, list[e] & 63, round_f32));
                atomicMax(&rowmax[rr], static_cast<unsigned long long>(__double_as_longlong(v)));
            }
        }
        __syncthreads();
        if (tid == 0) *lcount = 0u;
        const double am = __longlong_as_double(static_cast<long long>(rowmax[tid]));
        const double s = am / qmax;
        const float inv_s = static_cast<float>(qmax / am);
        const float qm = static_cast<float>(qmax);
        if (valid) (which ? sk : sq)[pair * L + r] = am == 0.0 ? 0.0 : s;
        __syncthreads();
        const float k1 = 1e-6f + 1.001f * rel, arow = dq * inv_s * 1.001f;
#pragma unroll
        for (int j = 0; j < KD; ++j) {
            float lv = 0.f;
            if (am != 0.0) {
                lv = cert_level(xv[j], arow * pn[j], k1, inv_s, qm);
                if (lv != lv) {
                    lv = 0.f;
                    if (valid) {
                        const unsigned slot = atomicAdd(lcount, 1u);
                        if (slot < kMaxList) {
                            list[slot] = (static_cast<uint32_t>(tid) << 6) | j;
                        } else {
                            const double xe = ref_chain_s<D, KD>(xa, tid, p, j, round_f32);
                            lv = static_cast<float>(fmin(fmax(round_half_away(xe / s), -qmax), qmax));
                        }
                    }
                }
            }
            lvl_s[tid * KD + j] = static_cast<uint16_t>(__float_as_uint(lv) >> 16);
        }
        __syncthreads();
        const unsigned n = min(*lcount, static_cast<unsigned>(kMaxList));
        for (unsigned e = tid; e < n; e += R) {
            const int rr = static_cast<int>(list[e] >> 6), j = static_cast<int>(list[e] & 63);
            const double sr = __longlong_as_double(static_cast<long long>(rowmax[rr])) / qmax;
            const double xe = ref_chain_s<D, KD>(xa, rr, p, j, round_f32);
            const float lv = static_cast<float>(fmin(fmax(round_half_away(xe / sr), -qmax), qmax));
            lvl_s[rr * KD + j] = static_cast<uint16_t>(__float_as_uint(lv) >> 16);
        }
        __syncthreads();
        if (valid) {
            uint16_t* out = (which ? lk : lq) + pair * L * KD;
            const uint4* src = reinterpret_cast<const uint4*>(lvl_s + tid * KD);
#pragma unroll
            for (int c = 0; c < KD / 8; ++c) *reinterpret_cast<uint4*>(out + lvl_index(L, r, c * 8)) = src[c];
        }
    } else {
    if (!QUANT && xhat != nullptr && valid) {
        // x^ and the row's bound factor for the streaming quantise pass:
        // [pair][tensor][L][KD] floats, then [pair][tensor][L] factors
        float* xo = xhat + ((pair * 2 + which) * L + r) * KD;
#pragma unroll
        for (int j = 0; j < KD; j += 4) *reinterpret_cast<float4*>(xo + j) = make_float4(xv[j], xv[j + 1], xv[j + 2], xv[j + 3]);
        xhat[gridDim.z * 2 * L * KD + (pair * 2 + which) * L + r] = dq;
    }
    if (!QUANT) {
        // e_j <= E_row = |q| d 2^-22 max_j |p_j| + rel max_j |x_j|: one bound per
        // row keeps the candidate test to a compare per element
        float xm = 0.f, pm = 0.f;
#pragma unroll
        for (int j = 0; j < KD; ++j) {
            xm = fmaxf(xm, fabsf(xv[j]));
            pm = fmaxf(pm, pn[j]);
        }
        const float er = fmaf(dq, pm, xm * rel) + 1e-30f;
        if (valid) atomicMax(red_f, __float_as_uint(fmaxf(0.f, (xm - er) * 0.999999f)));
        __syncthreads();
        const float thr = __uint_as_float(*red_f) - er;  // |x_j| >= LB - E_row
#pragma unroll
        for (int j = 0; j < KD; ++j)
            if (valid && fabsf(xv[j]) >= thr) {
                const unsigned slot = atomicAdd(lcount, 1u);
                if (slot < kMaxList) list[slot] = (static_cast<uint32_t>(tid) << 6) | j;
                else atomicMax(red_d, static_cast<unsigned long long>(__double_as_longlong(
                                          fabs(ref_chain_s<D, KD>(xa, tid, p, j, round_f32)))));
            }
        __syncthreads();
        const unsigned n = (DSA_ABLATE & 2048) ? 0u : min(*lcount, static_cast<unsigned>(kMaxList));  // profiling: no chains
#if DSA_ABLATE & 128
        if (tid == 0 && blockIdx.x % 8 == 3 && blockIdx.z == 5) printf("amax pass: tile %d tensor %d candidates %u\n", blockIdx.x, which, *lcount);
#endif
        double am = 0.0;
        for (unsigned e = tid; e < n; e += R)
            am = fmax(am, fabs(ref_chain_s<D, KD>(xa, static_cast<int>(list[e] >> 6), p, list[e] & 63, round_f32)));
        if (am > 0.0) atomicMax(red_d, static_cast<unsigned long long>(__double_as_longlong(am)));
        __syncthreads();
        if (tid == 0 && *red_d) atomicMax(amax + pair * 2 + which, *red_d);
    } else {
        const double am = __longlong_as_double(static_cast<long long>(amax[pair * 2 + which]));
        const double s = am / qmax;
        const float inv_s = static_cast<float>(qmax / am);
        const float qm = static_cast<float>(qmax);
        if (row0 == 0 && tid == 0) (which ? sk : sq)[pair] = am == 0.0 ? 0.0 : s;
        // certified levels -> staging; the rest -> shared list, recomputed
        // exactly by the whole CTA, then each thread writes its row
        const float k1 = 1e-6f + 1.001f * rel, arow = dq * inv_s * 1.001f;
#pragma unroll
        for (int j = 0; j < KD; ++j) {
            float lv = 0.f;
            if (am != 0.0) {
                lv = cert_level(xv[j], arow * pn[j], k1, inv_s, qm);
                if (lv != lv) {
                    lv = 0.f;
                    if (valid) {
                        const unsigned slot = atomicAdd(lcount, 1u);
                        if (slot < kMaxList) {
                            list[slot] = (static_cast<uint32_t>(tid) << 6) | j;
                        } else {
                            const double xe = ref_chain_s<D, KD>(xa, tid, p, j, round_f32);
                            lv = static_cast<float>(fmin(fmax(round_half_away(xe / s), -qmax), qmax));
                        }
                    }
                }
            }
            lvl_s[tid * KD + j] = static_cast<uint16_t>(__float_as_uint(lv) >> 16);
        }
        __syncthreads();
        const unsigned n = (DSA_ABLATE & 2048) ? 0u : min(*lcount, static_cast<unsigned>(kMaxList));  // profiling: no chains
#if DSA_ABLATE & 128
        if (tid == 0 && blockIdx.x % 8 == 3 && blockIdx.z == 5) printf("quant pass: tile %d tensor %d uncertified %u\n", blockIdx.x, which, *lcount);
#endif
        if (!round_f32) {
            // one thread per entry: split sum + certification, rarely the chain
            const double inv_s = qmax / am;
            for (unsigned e = tid; e < n; e += R) {
                const int rr = static_cast<int>(list[e] >> 6), j = static_cast<int>(list[e] & 63);
                const float lv = level_split<D, KD>(xa, rr, p, j, s, inv_s, qmax);
                lvl_s[rr * KD + j] = static_cast<uint16_t>(__float_as_uint(lv) >> 16);
            }
        } else {
            for (unsigned e = tid; e < n; e += R) {
                const int rr = static_cast<int>(list[e] >> 6), j = static_cast<int>(list[e] & 63);
                const double xe = ref_chain_s<D, KD>(xa, rr, p, j, round_f32);
                const float lv = static_cast<float>(fmin(fmax(round_half_away(xe / s), -qmax), qmax));
                lvl_s[rr * KD + j] = static_cast<uint16_t>(__float_as_uint(lv) >> 16);
            }
        }
        __syncthreads();
        if (valid) {
            uint16_t* out = (which ? lk : lq) + pair * L * KD;
            const uint4* src = reinterpret_cast<const uint4*>(lvl_s + tid * KD);
#pragma unroll
            for (int c = 0; c < KD / 8; ++c) *reinterpret_cast<uint4*>(out + lvl_index(L, r, c * 8)) = src[c];
        }
    }
    }  // !ROW
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<TC>(tmem);
}

// Streaming quantise pass over the stored x^ (thread = row x 8 columns):
// certified levels; the uncertified ones get list slots (one global atomic
// per warp that has any) and are recomputed by quantize_fix_kernel, one thread each
// (in place, by the reference chain, only if the list is full).
template <int D, int KD>
__global__ void __launch_bounds__(256)
    quantize_xhat_kernel(const float* xhat, const __nv_bfloat16* __restrict__ q,
                         const __nv_bfloat16* __restrict__ k, const float* __restrict__ p,
                         const unsigned char* __restrict__ img, int64_t pairs, int64_t L, int round_f32,
                         double qmax, const unsigned long long* __restrict__ amax, uint16_t* __restrict__ lq,
                         uint16_t* __restrict__ lk, double* __restrict__ sq, double* __restrict__ sk) {
    using Sm = ProjSmem<D, KD>;
    constexpr int NC = KD / 8;
    // grid = (ceil(L * NC / 256), pairs * 2): one tensor per blockIdx.y, so
    // its scale is computed once per block (no 64-bit division per thread)
    const int64_t pw = blockIdx.y;  // pair * 2 + which
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    __shared__ double s_s;
    __shared__ float s_inv;
    if (threadIdx.x == 0) {
        const double am0 = __longlong_as_double(static_cast<long long>(amax[pw]));
        s_s = am0 / qmax;
        s_inv = static_cast<float>(qmax / am0);
    }
    __syncthreads();
    // no early exit before the warp-wide slot allocation below
    const bool active = idx < L * NC;
    const int c = static_cast<int>(idx % NC);
    const int64_t r = active ? idx / NC : 0;
    const int64_t rr = pw * L + r;  // (pair * 2 + which) * L + r
    const int which = static_cast<int>(pw & 1);
    const int64_t pair = pw >> 1;
    const double am = __longlong_as_double(static_cast<long long>(amax[pw]));
    const double s = s_s;
    if (active && r == 0 && c == 0) (which ? sk : sq)[pair] = am == 0.0 ? 0.0 : s;
    const float inv_s = s_inv;
    const float qm = static_cast<float>(qmax);
    const float rel = round_f32 ? 2.4e-7f : 1.2e-7f;
    const float* pn = reinterpret_cast<const float*>(img + Sm::kB);
    // deferred list: counter then entries after the bound factors
    unsigned long long* lcnt = reinterpret_cast<unsigned long long*>(const_cast<float*>(xhat) + pairs * 2 * L * (KD + 1));
    unsigned long long* list = lcnt + 1;
    const int64_t lcap = pairs * L * KD / 4;
    float xv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float dq = 0.f;
    if (active) {
        const float4 a0 = __ldg(reinterpret_cast<const float4*>(xhat + rr * KD + c * 8));
        const float4 a1 = __ldg(reinterpret_cast<const float4*>(xhat + rr * KD + c * 8 + 4));
        dq = __ldg(xhat + pairs * 2 * L * KD + rr);
        xv[0] = a0.x; xv[1] = a0.y; xv[2] = a0.z; xv[3] = a0.w;
        xv[4] = a1.x; xv[5] = a1.y; xv[6] = a1.z; xv[7] = a1.w;
    }
    const float k1 = 1e-6f + 1.001f * rel, arow = dq * inv_s * 1.001f;
    float lv[8];
    unsigned um = 0;  // uncertified columns of this thread
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        lv[u] = 0.f;
        if (active && am != 0.0) {
            lv[u] = cert_level(xv[u], arow * __ldg(pn + c * 8 + u), k1, inv_s, qm);
            if (lv[u] != lv[u]) {
                lv[u] = 0.f;
                um |= 1u << u;
            }
        }
    }
    // warp-aggregated slot allocation: uncertified levels are rare (~0.04 %),
    // so almost every warp skips the atomic and no block barrier is needed
    const int lane = threadIdx.x & 31;
    const unsigned cnt = static_cast<unsigned>(__popc(um));
    unsigned long long slot = 0;
    if (__any_sync(0xffffffffu, cnt != 0)) {
        unsigned incl = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long base = 0;
        if (lane == 31) base = atomicAdd(lcnt, static_cast<unsigned long long>(tot));
        base = __shfl_sync(0xffffffffu, base, 31);
        slot = base + (incl - cnt);
    }
    while (um) {
        const int u = __ffs(um) - 1;
        um &= um - 1u;
        const int j = c * 8 + u;
        if (slot < static_cast<unsigned long long>(lcap)) {
            list[slot] = (static_cast<unsigned long long>(pw) << 40) | (static_cast<unsigned long long>(r) << 6) |
                         static_cast<unsigned long long>(j);
        } else {  // list full: the reference chain in place
            const __nv_bfloat16* row = (which ? k : q) + (pair * L + r) * D;
            double acc = 0.0;
            for (int t = 0; t < D; ++t) acc = fma(to_double(row[t]), static_cast<double>(__ldg(p + t * KD + j)), acc);
            if (round_f32) acc = static_cast<double>(static_cast<float>(acc));
            lv[u] = static_cast<float>(fmin(fmax(round_half_away(acc / s), -qmax), qmax));
        }
        ++slot;
    }
    if (!active) return;
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h)
        w[h] = (__float_as_uint(lv[2 * h]) >> 16) | ((__float_as_uint(lv[2 * h + 1]) >> 16) << 16);
    uint16_t* out = (which ? lk : lq) + pair * L * KD;
    *reinterpret_cast<uint4*>(out + lvl_index(L, r, c * 8)) = make_uint4(w[0], w[1], w[2], w[3]);
}

// The levels quantize_xhat_kernel could not certify: one thread per list
// entry runs the reference's fp64 chain (P/src/kernels/scalar.cpp:19-32) and
// overwrites the placeholder level.
template <int D, int KD>
__global__ void __launch_bounds__(256)
    quantize_fix_kernel(const float* __restrict__ xhat, const __nv_bfloat16* __restrict__ q,
                        const __nv_bfloat16* __restrict__ k, const float* __restrict__ p, int64_t pairs, int64_t L,
                        int round_f32, double qmax, const unsigned long long* __restrict__ amax,
                        uint16_t* __restrict__ lq, uint16_t* __restrict__ lk) {
    const unsigned long long* lcnt =
        reinterpret_cast<const unsigned long long*>(xhat + pairs * 2 * L * (KD + 1));
    const unsigned long long* list = lcnt + 1;
    // P (exact f32 -> f64) staged in shared memory, so the 64- / 128-step
    // chain below waits on FMAs only, not on a load per step; its loads are
    // issued alongside the list-count read
    __shared__ double ps[D * KD];
    const int64_t n = min(static_cast<int64_t>(*lcnt), pairs * L * KD / 4);
    for (int i = threadIdx.x; i < D * KD; i += blockDim.x) ps[i] = static_cast<double>(__ldg(p + i));
    if (static_cast<int64_t>(blockIdx.x) * blockDim.x >= n) return;  // the list is short: most blocks idle
    __syncthreads();
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long v = list[e];
        const int64_t pw = static_cast<int64_t>(v >> 40), r = static_cast<int64_t>((v >> 6) & 0x3ffffffffull);
        const int j = static_cast<int>(v & 63);
        const int which = static_cast<int>(pw & 1);
        const int64_t pair = pw >> 1;
        const double s = __longlong_as_double(static_cast<long long>(amax[pw])) / qmax;
        const uint4* row = reinterpret_cast<const uint4*>((which ? k : q) + (pair * L + r) * D);
        uint4 xr[D / 8];
#pragma unroll
        for (int t = 0; t < D / 8; ++t) xr[t] = __ldg(row + t);  // the whole row in flight at once
        const __nv_bfloat16* xe = reinterpret_cast<const __nv_bfloat16*>(xr);
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < D; ++t) acc = fma(to_double(xe[t]), ps[t * KD + j], acc);
        if (round_f32) acc = static_cast<double>(static_cast<float>(acc));
        const float lv = static_cast<float>(fmin(fmax(round_half_away(acc / s), -qmax), qmax));
        (which ? lk : lq)[pair * L * KD + lvl_index(L, r, j)] = static_cast<uint16_t>(__float_as_uint(lv) >> 16);
    }
}

template <int D, int KD, int R>
void launch_tc(const PredictArgs& a, cudaStream_t st) {
    using Sm = ProjSmem<D, KD, R>;
    constexpr int N = 3 * KD;
    constexpr int TC = (R / 128) * N <= 64 ? 64 : ((R / 128) * N <= 128 ? 128 : 256);
    // no more CTAs per SM than TMEM holds (512 columns)
    const int smem = std::max(Sm::bytes(), (228 * 1024) / (512 / TC + 1) + 1024);
    auto ka = project_tc_kernel<D, KD, false, R>;
    auto kq = project_tc_kernel<D, KD, true, R>;
    cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const auto* q = static_cast<const __nv_bfloat16*>(a.q);
    const auto* k = static_cast<const __nv_bfloat16*>(a.k);
    const dim3 grid(static_cast<unsigned>(ceil_div_i(a.L, R)), 2, static_cast<unsigned>(a.pairs));
    unsigned long long* lcnt =
        a.xhat != nullptr && !a.per_row ? reinterpret_cast<unsigned long long*>(a.xhat + a.pairs * 2 * a.L * (KD + 1)) : nullptr;
    psplit_kernel<D, KD><<<1, 256, 0, st>>>(a.p, a.pimg, a.per_row ? nullptr : a.amax, 2 * a.pairs, lcnt);
    if (a.per_row) {
        auto kr = project_tc_kernel<D, KD, true, R, true>;
        const int rsmem = std::max(ProjSmem<D, KD, R, true>::bytes(), (228 * 1024) / (512 / TC + 1) + 1024);
        cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, rsmem);
        kr<<<grid, R, rsmem, st>>>(q, k, a.p, a.pimg, a.L, a.round_f32, a.qmax, nullptr, a.lq, a.lk, a.sq, a.sk,
                                  nullptr);
        note_launch(2);
        return;
    }
    if (a.xhat != nullptr) {
        // amax pass stores x^ (fp32) + bound factors; the quantise pass streams them
        ka<<<grid, R, smem, st>>>(q, k, a.p, a.pimg, a.L, a.round_f32, a.qmax, a.amax, a.lq, a.lk, a.sq, a.sk,
                                  a.xhat);
        const dim3 gq(static_cast<unsigned>(ceil_div_i(a.L * (KD / 8), 256)), static_cast<unsigned>(a.pairs * 2));
        quantize_xhat_kernel<D, KD><<<gq, 256, 0, st>>>(
            a.xhat, q, k, a.p, a.pimg, a.pairs, a.L, a.round_f32, a.qmax, a.amax, a.lq, a.lk, a.sq, a.sk);
        quantize_fix_kernel<D, KD><<<2 * sm_count(), 256, 0, st>>>(a.xhat, q, k, a.p, a.pairs, a.L, a.round_f32, a.qmax,
                                                           a.amax, a.lq, a.lk);
        note_launch();
    } else {
        ka<<<grid, R, smem, st>>>(q, k, a.p, a.pimg, a.L, a.round_f32, a.qmax, a.amax, a.lq, a.lk, a.sq, a.sk,
                                  nullptr);
        kq<<<grid, R, smem, st>>>(q, k, a.p, a.pimg, a.L, a.round_f32, a.qmax, a.amax, a.lq, a.lk, a.sq, a.sk,
                                  nullptr);
    }
    note_launch(3);
}

template <int D, int KD>
void launch_tc(const PredictArgs& a, cudaStream_t st) {
    // d = 128: 256 rows per CTA (two M = 128 MMAs share the P image and prologue)
    if (D == 128 && !(DSA_ABLATE & 1024)) launch_tc<D, KD, 256>(a, st);
    else launch_tc<D, KD, 128>(a, st);
}

}  // namespace

size_t predict_tc_image_bytes(int64_t D, int64_t KD) { return static_cast<size_t>(3 * KD * D * 2 + KD * 4); }

bool predict_tc_supported(const PredictArgs& a) {
    if (!a.bf16 || a.pimg == nullptr) return false;
    return (a.D == 64 || a.D == 128) && (a.KD == 16 || a.KD == 32);
}

void run_predict_tc(const PredictArgs& a, cudaStream_t st) {
    if (a.D == 64) {
        if (a.KD == 16) launch_tc<64, 16>(a, st);
        else launch_tc<64, 32>(a, st);
    } else {
        if (a.KD == 16) launch_tc<128, 16>(a, st);
        else launch_tc<128, 32>(a, st);
    }
}

}  // namespace dsa
