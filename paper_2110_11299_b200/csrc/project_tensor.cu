// Projection + per-tensor quantisation in ONE pass over Q/K: one CTA per
// (pair, tensor) for the d = 64, k = 16 shapes with L <= 4096 (C2-class).
//
// Reference semantics: x = q . P by the sequential fp64 FMA
// chain of P/src/kernels/scalar.cpp:19-32, amax over the whole tensor, s =
// amax / qmax, level = round-half-away(x / s) (scalar.cpp:11-17).  The
// arithmetic is the one project_tc.cu certifies (exact three-way bf16 split
// of P on tcgen05, fp32 accumulation, per-element error bound, fp64 chains
// for the candidates of the maximum and for the uncertified levels); what
// changes is the schedule.  The tile kernels need the tensor's amax before
// any level, so they either read Q/K twice or round-trip x^ through HBM
// (read X 128 B + write/read x^ 2 x 64 B + levels 32 B per row).  Here the
// whole tensor's x^ stays on chip -- 26 of 32 tiles in TMEM (16 columns
// each, written back with tcgen05.st), the rest in shared memory -- so HBM
// sees X once and the levels once (160 B per row), and psplit /
// quantise / fix-up launches disappear (the P image is built in the
// prologue, the amax is CTA-local).
//
// Warp roles (448 threads, one CTA per SM: TMEM 512 columns):
//   warp 8 (one lane): TMA 2-D loads of 128-row X tiles (128 B rows,
//     SWIZZLE_128B) into a 6-stage ring, full/empty mbarriers;
//   warp 9 (one lane): per tile, X . [P1|P2|P3] (M = 128, N = 48, K = 64) into
//     one of two 48-column accumulator slots;
//   warps 0-7: group g = warp / 4 takes tiles t = g (mod 2): the row's |q|
//     (bound factor) from the staged tile, drain of slot g, x^ = P1 part +
//     (P2 part + P3 part), x^ parked in TMEM / shared memory, running lower
//     bound of the maximum.  Then: candidates of the maximum -> exact chains ->
//     amax; certified levels stored, uncertified ones recomputed.
#include <cuda.h>
#include <cuda_bf16.h>

#include <climits>

#include "device_common.cuh"
#include "kernels.h"
#include "tc_sm100.cuh"
#include "tma_map.h"

namespace dsa {
namespace {

// Profiling-only build (-DDSA_PT_PROBE, tools/pt_probe.py): %globaltimer
// at the phase boundaries of every CTA.  Never in the product library.
#ifdef DSA_PT_PROBE
__device__ unsigned long long g_pt_probe[4096][8];
__device__ unsigned g_pt_count[4096][2];
#define PT_COUNT(i) atomicAdd(&g_pt_count[blockIdx.x & 4095][i], 1u)
#define PT_PROBE(i)                                                                               \
    do {                                                                                          \
        if (threadIdx.x == 0) {                                                                   \
            unsigned long long t_;                                                                \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                \
            g_pt_probe[blockIdx.x & 4095][i] = t_;                                                \
            if ((i) == 1) {                                                                       \
                unsigned sm_;                                                                     \
                asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));                                  \
                g_pt_probe[blockIdx.x & 4095][7] = sm_;                                           \
            }                                                                                     \
        }                                                                                         \
    } while (0)
#else
#define PT_COUNT(i) \
    do {            \
    } while (0)
#define PT_PROBE(i) \
    do {            \
    } while (0)
#endif

constexpr int kThreads = 448;  // 8 drain warps, TMA warp, MMA warp, 4 norm warps

template <int D, int KD>
struct TensorSmem {
    static constexpr int N = 3 * KD;                      // MMA N: P1 | P2 | P3
    static constexpr int kStages = 6;
    static constexpr int kTile = 128 * D * 2;             // one 128-row X tile
    static constexpr int kTmemTiles = (512 - 2 * N) / KD; // x^ tiles parked in TMEM
    static constexpr int kMaxTiles = 32;                  // L <= 4096
    static constexpr int kSmemTiles = kMaxTiles > kTmemTiles ? kMaxTiles - kTmemTiles : 0;
    static constexpr int kList = 2048;                    // (row, column) entries for the fp64 chains
    static constexpr int oRing = 0;
    static constexpr int oXs = oRing + kStages * kTile;
    static constexpr int oImg = oXs + kSmemTiles * 128 * KD * 4;
    static constexpr int oPn = oImg + N * D * 2;
    static constexpr int oPd = oPn + 256;
    static constexpr int oDq = oPd + D * KD * 8;
    static constexpr int oList = oDq + kMaxTiles * 128 * 4;
    static constexpr int oBar = oList + kList * 4;
    static constexpr int oMisc = oBar + (2 * kStages + 4) * 8;
    static constexpr int oReady = oMisc + 64;                  // per tile: norm warps done
    static constexpr int bytes = oReady + kMaxTiles * 4;
};

// K-major no-swizzle operand layout (the P image, as in project_tc.cu)
template <int D>
__device__ __forceinline__ uint32_t img_off(int r, int c) {
    return static_cast<uint32_t>((r >> 3) * (D * 16) + (c >> 3) * 128 + (r & 7) * 16 + (c & 7) * 2);
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// the reference's fp64 chain (scalar.cpp:19-32) for row `row` of X, P in
// f64 from shared memory.  Out of line: it is latency-bound (64 dependent
// DFMAs) and rare, and inlined copies would bloat the kernel's code.
template <int D, int KD>
__device__ __noinline__ double chain_g(const __nv_bfloat16* __restrict__ row, const double* pd, int j,
                                       int round_f32) {
    uint4 xr[D / 8];  // the whole row in flight at once
#pragma unroll
    for (int c = 0; c < D / 8; ++c) xr[c] = __ldg(reinterpret_cast<const uint4*>(row) + c);
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < D / 8; ++c) {
        const __nv_bfloat16* xe = reinterpret_cast<const __nv_bfloat16*>(&xr[c]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fma(to_double(xe[u]), pd[(c * 8 + u) * KD + j], acc);
    }
    return round_f32 ? static_cast<double>(static_cast<float>(acc)) : acc;
}

template <int D, int KD>
__global__ void __launch_bounds__(kThreads, 1)
    project_tensor_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                          const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                          const float* __restrict__ p, int64_t L, int round_f32, double qmax,
                          uint16_t* __restrict__ lq, uint16_t* __restrict__ lk, double* __restrict__ sq,
                          double* __restrict__ sk) {
    static_assert(D == 64, "one 128-byte swizzled row per X row");
    static_assert(KD == 16, "x^ tile = 16 TMEM columns");
    using Sm = TensorSmem<D, KD>;
    constexpr int N = Sm::N, S = Sm::kStages, kTT = Sm::kTmemTiles;
    // no static shared memory in this kernel: the dynamic window starts at
    // the CTA's shared base (1024-byte aligned, as SWIZZLE_128B needs); kept
    // as a __shared__ array so every access compiles to LDS / STS
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* ring = sm + Sm::oRing;
    float4* xs4 = reinterpret_cast<float4*>(sm + Sm::oXs);
    unsigned char* img = sm + Sm::oImg;
    float* pn = reinterpret_cast<float*>(sm + Sm::oPn);
    double* pd = reinterpret_cast<double*>(sm + Sm::oPd);
    float* dq_s = reinterpret_cast<float*>(sm + Sm::oDq);
    uint32_t* list = reinterpret_cast<uint32_t*>(sm + Sm::oList);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + Sm::oBar);
    uint64_t* empty = full + S;
    uint64_t* accf = full + 2 * S;  // [2]
    uint64_t* acce = accf + 2;      // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + Sm::oMisc);
    unsigned* lb_u = tslot + 1;
    unsigned* cnt = tslot + 2;  // [2]
    unsigned long long* am_u = reinterpret_cast<unsigned long long*>(sm + Sm::oMisc + 16);
    unsigned* ready = reinterpret_cast<unsigned*>(sm + Sm::oReady);

    PT_PROBE(0);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int which = static_cast<int>(blockIdx.x & 1);
    const int64_t pair = blockIdx.x >> 1;
    const int T = static_cast<int>((L + 127) / 128);
    const __nv_bfloat16* X = (which ? k : q) + pair * L * D;
    const CUtensorMap* map = which ? &mk : &mq;
    auto load_tile = [&](int t) {
        const int s = t % S;
        tc::mbar_expect_tx(&full[s], Sm::kTile);
        tc::tma_load_2d(tc::smem_addr(ring + s * Sm::kTile), map, 0, static_cast<int>(pair * L + t * 128), &full[s]);
    };
    if (warp == 8 && lane == 0) {
        // barriers, then the first ring's worth of X tiles in flight while
        // the rest of the CTA builds the P image
        for (int s = 0; s < S; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1 + 4);  // MMA commit + the 4 norm warps
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&accf[a], 1);
            tc::mbar_init(&acce[a], 4);
        }
        tc::fence_barrier_init();
        for (int t = 0; t < min(S, T); ++t) load_tile(t);
    }

    // prologue: P split exactly into three bf16 parts (B-operand image) and
    // P in f64 for the chains
    constexpr int kPer = (D * KD + kThreads - 1) / kThreads;
    float pv[kPer];  // all of this thread's P loads in flight at once
#pragma unroll
    for (int m = 0; m < kPer; ++m) pv[m] = tid + m * kThreads < D * KD ? __ldg(p + tid + m * kThreads) : 0.f;
#pragma unroll
    for (int m = 0; m < kPer; ++m) {
        const int i = tid + m * kThreads;
        if (i >= D * KD) break;
        const int c = i / KD, j = i % KD;
        const float v = pv[m];
        pd[i] = static_cast<double>(v);
        const __nv_bfloat16 b1 = __float2bfloat16_rn(v);
        const float r1 = v - __bfloat162float(b1);
        const __nv_bfloat16 b2 = __float2bfloat16_rn(r1);
        const float r2 = r1 - __bfloat162float(b2);
        *reinterpret_cast<__nv_bfloat16*>(img + img_off<D>(j, c)) = b1;
        *reinterpret_cast<__nv_bfloat16*>(img + img_off<D>(KD + j, c)) = b2;
        *reinterpret_cast<__nv_bfloat16*>(img + img_off<D>(2 * KD + j, c)) = __float2bfloat16_rn(r2);
    }
    if (tid < Sm::kMaxTiles) ready[tid] = 0u;
    if (tid == 0) {
        *lb_u = 0u;
        cnt[0] = cnt[1] = 0u;
        *am_u = 0ull;
    }
    if (warp == 9) tc::tmem_alloc<512>(tslot);
    tc::fence_proxy_async();  // the P image (generic stores) -> the MMA's async proxy
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tslot;
    PT_PROBE(1);
    const float rel = round_f32 ? 2.4e-7f : 1.2e-7f;

    if (warp == 8) {
        if (lane == 0) {
            for (int t = S; t < T; ++t) {
                tc::mbar_wait(&empty[t % S], ((t / S) & 1) ^ 1);
                load_tile(t);
            }
        }
    } else if (warp == 9) {
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_bf16_f32(128, N);
            const uint32_t bs = tc::smem_addr(img);
            for (int t = 0; t < T; ++t) {
                const int s = t % S, a = t & 1;
                tc::mbar_wait(&full[s], (t / S) & 1);
                tc::mbar_wait(&acce[a], ((t >> 1) & 1) ^ 1);
                tc::fence_after_sync();
                const uint32_t xs = tc::smem_addr(ring + s * Sm::kTile);
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint64_t ad = tc::desc_sw128(xs + ks * 32, 16, 1024);
                    const uint64_t bd = tc::desc_kmajor_nosw(bs + ks * 256, 128, D * 16);
                    tc::mma_bf16(tmem + a * N, ad, bd, idesc, ks > 0);
                }
                tc::commit(&accf[a]);
                tc::commit(&empty[s]);
            }
        }
    } else if (warp >= 10) {
        // norm warps: |q| of every row (Cauchy-Schwarz partner of |p_j|)
        // from the swizzled tile (16-byte chunk c of row r at r * 128 + ((c ^
        // (r & 7)) * 16)): bf16 pairs widened by a shift / mask, packed FFMA2.
        // Off the drain warps' critical path; they run ahead, gated by TMA.
        const int rr = (warp - 10) * 32 + lane;
        for (int t = 0; t < T; ++t) {
            const int s = t % S;
            tc::mbar_wait(&full[s], (t / S) & 1);
            const unsigned char* tile = ring + s * Sm::kTile;
            float2 a2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int ch = 0; ch < D / 8; ++ch) {
                const uint4 v = *reinterpret_cast<const uint4*>(tile + rr * 128 + ((ch ^ (rr & 7)) << 4));
                const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2 f = make_float2(__uint_as_float(wv[u] << 16), __uint_as_float(wv[u] & 0xffff0000u));
                    a2 = __ffma2_rn(f, f, a2);
                }
            }
            dq_s[t * 128 + rr] =
                (sqrtf(a2.x + a2.y) * 1.001f + 1e-30f) * (static_cast<float>(D) * 2.384185791015625e-7f);
            __syncwarp();
            if (lane == 0) {
                tc::mbar_arrive(&empty[s]);  // the stage is free once |q| is read
                __threadfence_block();
                atomicAdd(&ready[t], 1u);
            }
        }
    } else {
        // streaming: warp group g drains the tiles t = g (mod 2)
        const int g = warp >> 2, rr = (warp & 3) * 32 + lane;
        const uint32_t lanes = static_cast<uint32_t>((warp & 3) * 32) << 16;
        // max_j |p_j| 1.001 (bound factor), per warp while its first tile is
        // in flight: lane = (column l % 16, rows of half l / 16)
        float pm;
        {
            double s2 = 0.0;
            const int j = lane & (KD - 1), h = lane / KD;
#pragma unroll 8
            for (int u = h * (D / 2); u < (h + 1) * (D / 2); ++u) s2 = fma(pd[u * KD + j], pd[u * KD + j], s2);
            s2 += __shfl_xor_sync(0xffffffffu, s2, KD);
            float v = static_cast<float>(sqrt(s2) * 1.001);
#pragma unroll
            for (int o = KD / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
            pm = v;
            if (warp == 0 && lane < KD) pn[lane] = static_cast<float>(sqrt(s2) * 1.001);
        }
        float lb = 0.f;
        for (int t = g; t < T; t += 2) {
            tc::mbar_wait(&accf[g], (t >> 1) & 1);
            tc::fence_after_sync();
            uint32_t d0[32], d1[16];
            tc::ld_32x32b_x32(tmem + lanes + g * N, d0);
            tc::ld_32x32b_x16(tmem + lanes + g * N + 32, d1);
            tc::wait_ld();
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&acce[g]);
            uint32_t xb[KD];
            float xm = 0.f;
#pragma unroll
            for (int j = 0; j < KD; ++j) {
                const float x = __uint_as_float(d0[j]) + (__uint_as_float(d0[16 + j]) + __uint_as_float(d1[j]));
                xb[j] = __float_as_uint(x);
                xm = fmaxf(xm, fabsf(x));
            }
            if (t < kTT) {
                tc::st_32x32b_x16(tmem + lanes + 2 * N + t * KD, xb);
            } else {
#pragma unroll
                for (int jq = 0; jq < KD / 4; ++jq)
                    xs4[((t - kTT) * (KD / 4) + jq) * 128 + rr] =
                        make_float4(__uint_as_float(xb[4 * jq]), __uint_as_float(xb[4 * jq + 1]),
                                    __uint_as_float(xb[4 * jq + 2]), __uint_as_float(xb[4 * jq + 3]));
            }
            // e_j <= E_row = dq max_j |p_j| + rel max_j |x_j| (as project_tc.cu);
            // dq from the norm warps (tile-indexed flag, no phase aliasing)
            while (*reinterpret_cast<volatile unsigned*>(&ready[t]) < 4u) __nanosleep(32);
            __threadfence_block();
            const float dq = dq_s[t * 128 + rr];
            const float er = fmaf(dq, pm, xm * rel) + 1e-30f;
            const int64_t row = static_cast<int64_t>(t) * 128 + rr;
            const bool valid = row < L;
            // candidates of the maximum, against the running lower bound LB_t
            // (this warp's tile, every tile published so far): LB_t <= the
            // final LB, so every final candidate (|x^_j| >= LB - E_row) is
            // caught here (its X row re-read from L2, where the tile's TMA
            // load just passed); the exact chains' maximum is the amax
            float lbw = valid ? fmaxf(0.f, (xm - er) * 0.999999f) : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) lbw = fmaxf(lbw, __shfl_xor_sync(0xffffffffu, lbw, o));
            lb = fmaxf(lb, lbw);
            if (lane == 0) atomicMax(lb_u, __float_as_uint(lb));
            const float thr = fmaxf(lb, __uint_as_float(*reinterpret_cast<volatile unsigned*>(lb_u))) - er;
            const bool cand = valid && xm >= thr;
            if (__any_sync(0xffffffffu, cand) && cand) {
#pragma unroll  // xb stays in registers (a rolled loop would index it dynamically)
                for (int j = 0; j < KD; ++j) {
                    const float ax = fabsf(__uint_as_float(xb[j]));
                    if (ax < thr) continue;
                    PT_COUNT(0);
                    // (row, column) and |x^_j| + E_row: the final test is
                    // |x^_j| + E_row >= LB after the last tile
                    const unsigned slot = atomicAdd(&cnt[0], 1u);
                    if (slot < Sm::kList / 2) {
                        list[2 * slot] = (static_cast<uint32_t>(row) << 6) | j;
                        list[2 * slot + 1] = __float_as_uint(ax + er);
                        prefetch_l1(X + row * D);
                    } else {
                        atomicMax(am_u, static_cast<unsigned long long>(__double_as_longlong(
                                            fabs(chain_g<D, KD>(X + row * D, pd, j, round_f32)))));
                    }
                }
            }
        }
        tc::wait_st();
    }
    tc::fence_before_sync();
    __syncthreads();
    PT_PROBE(2);
    tc::fence_after_sync();

    PT_PROBE(3);
    {
        // the recorded candidates that pass the final bound, one chain each
        const unsigned n = min(cnt[0], static_cast<unsigned>(Sm::kList / 2));
        const float LB = __uint_as_float(*lb_u);
        for (unsigned e = tid; e < n; e += blockDim.x)
            if (__uint_as_float(list[2 * e + 1]) >= LB)
                atomicMax(am_u, static_cast<unsigned long long>(__double_as_longlong(fabs(chain_g<D, KD>(
                                    X + static_cast<int64_t>(list[2 * e] >> 6) * D, pd, list[2 * e] & 63, round_f32)))));
    }
    __syncthreads();
    PT_PROBE(4);
    const double am = __longlong_as_double(static_cast<long long>(*am_u));
    const double s = am / qmax;
    if (tid == 0) (which ? sk : sq)[pair] = am == 0.0 ? 0.0 : s;
    uint16_t* out = (which ? lk : lq) + pair * L * KD;

    // levels: t = x^ / s is certified when |t - rint(t)| + margin < 1/2
    // (margin_j = |t| K1 + B_j as in project_tc.cu's cert_level); a certified
    // level is rint(t): t is away from every .5 boundary, where round-half-
    // away = round-to-nearest, and |t| < qmax + 1/2, so the reference's clamp
    // is inactive.  Per element: packed FFMA2 (x/s + 1.5 2^23 -> the nearest
    // integer), FADD2 (the integer), FFMA2 (x/s - integer), a max; ONE test
    // per row against the row's largest margin (|t| <= qmax + 1/2, p_j <=
    // max_j p_j); in a row that fails it, the elements past that margin
    // are recomputed by the reference chain.
    // The level keeps the sign of x (the reference's trunc gives -0).
    if (warp < 8) {
        const int g = warp >> 2, rr = (warp & 3) * 32 + lane;
        const float inv_s = static_cast<float>(qmax / am);
        const float k1 = 1e-6f + 1.001f * rel;
        float pm = 0.f;
#pragma unroll
        for (int j = 0; j < KD; ++j) pm = fmaxf(pm, pn[j]);
        const float kq = static_cast<float>(qmax + 0.5) * k1;
        const float2 inv2 = make_float2(inv_s, inv_s);
        const float2 mg2 = make_float2(12582912.f, 12582912.f);
        const float2 nmg2 = make_float2(-12582912.f, -12582912.f);
        // four tiles per step: their TMEM loads in flight together
        constexpr int kB = 4;
        for (int t0 = g; t0 < T; t0 += 2 * kB) {
            uint32_t xb[kB][KD];
            float dqb[kB];
#pragma unroll
            for (int bi = 0; bi < kB; ++bi) {
                const int t = t0 + 2 * bi;
                if (t >= T) break;  // warp-uniform
                dqb[bi] = dq_s[t * 128 + rr];
                if (t < kTT) {
                    tc::ld_32x32b_x16(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 2 * N + t * KD, xb[bi]);
                } else {
#pragma unroll
                    for (int jq = 0; jq < KD / 4; ++jq) {
                        const float4 v = xs4[((t - kTT) * (KD / 4) + jq) * 128 + rr];
                        xb[bi][4 * jq] = __float_as_uint(v.x);
                        xb[bi][4 * jq + 1] = __float_as_uint(v.y);
                        xb[bi][4 * jq + 2] = __float_as_uint(v.z);
                        xb[bi][4 * jq + 3] = __float_as_uint(v.w);
                    }
                }
            }
            tc::wait_ld();
#pragma unroll
            for (int bi = 0; bi < kB; ++bi)
#pragma unroll
                for (int j = 0; j < KD; ++j) asm volatile("" : "+r"(xb[bi][j]));  // no use before the wait
#pragma unroll
            for (int bi = 0; bi < kB; ++bi) {
                const int t = t0 + 2 * bi;
                if (t >= T) break;
                const int64_t row = static_cast<int64_t>(t) * 128 + rr;
                if (row >= L) continue;
                float xv[KD];
#pragma unroll
                for (int j = 0; j < KD; ++j) xv[j] = __uint_as_float(xb[bi][j]);
                const float arow = dqb[bi] * inv_s * 1.001f;
                uint32_t w[KD / 2];
                float dv[KD];
                float dmax = 0.f;
#pragma unroll
                for (int h = 0; h < KD / 2; ++h) {
                    const float2 x2 = make_float2(xv[2 * h], xv[2 * h + 1]);
                    const float2 b = __ffma2_rn(x2, inv2, mg2);
                    const float2 r = __fadd2_rn(b, nmg2);
                    const float2 d = __ffma2_rn(x2, inv2, make_float2(-r.x, -r.y));
                    dv[2 * h] = d.x;
                    dv[2 * h + 1] = d.y;
                    dmax = fmaxf(dmax, fmaxf(fabsf(d.x), fabsf(d.y)));
                    const uint32_t lo = __float_as_uint(r.x) | (__float_as_uint(x2.x) & 0x80000000u);
                    const uint32_t hi = __float_as_uint(r.y) | (__float_as_uint(x2.y) & 0x80000000u);
                    w[h] = __byte_perm(lo, hi, 0x7632);
                }
                if (am == 0.0) {
#pragma unroll
                    for (int h = 0; h < KD / 2; ++h) w[h] = 0u;
                }
#pragma unroll
                for (int c = 0; c < KD / 8; ++c)
                    *reinterpret_cast<uint4*>(out + lvl_index(L, row, c * 8)) =
                        make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
                // the row's largest margin: |t| <= qmax + 1/2, p_j <= max_j p_j.
                // Rare: the elements past it are listed (their stored level is
                // overwritten after the barrier by the reference chain), or
                // recomputed here once the list is full.
                const float dthr = 0.5f - fmaf(arow, pm, kq);
                if (dmax >= dthr && am != 0.0) {
                    PT_COUNT(1);
                    unsigned um = 0;
#pragma unroll
                    for (int j = 0; j < KD; ++j) um |= (fabsf(dv[j]) >= dthr ? 1u : 0u) << j;
#pragma unroll 1
                    while (um) {
                        const int j = __ffs(um) - 1;
                        um &= um - 1u;
                        const unsigned slot = atomicAdd(&cnt[1], 1u);
                        if (slot < Sm::kList) {
                            list[slot] = (static_cast<uint32_t>(row) << 6) | j;
                            prefetch_l1(X + row * D);  // the chain after the barrier reads it from L1
                        } else {
                            const double xe = chain_g<D, KD>(X + row * D, pd, j, round_f32);
                            const float lv = static_cast<float>(fmin(fmax(round_half_away(xe / s), -qmax), qmax));
                            out[lvl_index(L, row, j)] = static_cast<uint16_t>(__float_as_uint(lv) >> 16);
                        }
                    }
                }
            }
        }
    }
    __syncthreads();
    PT_PROBE(5);
    {
        const unsigned n = min(cnt[1], static_cast<unsigned>(Sm::kList));
        for (unsigned e = tid; e < n; e += blockDim.x) {
            const int64_t row = static_cast<int64_t>(list[e] >> 6);
            const int j = static_cast<int>(list[e] & 63);
            const double xe = chain_g<D, KD>(X + row * D, pd, j, round_f32);
            const float lv = static_cast<float>(fmin(fmax(round_half_away(xe / s), -qmax), qmax));
            out[lvl_index(L, row, j)] = static_cast<uint16_t>(__float_as_uint(lv) >> 16);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    PT_PROBE(6);
    if (warp == 9) tc::tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------
// Two-read variant (tensors whose x^ does not fit on chip: d = 128 / k = 32
// (C3), or L > 4096): the same CTA per (pair, tensor) streams its tensor
// TWICE through the tensor core -- pass A the exact amax (candidates of the
// maximum -> fp64 chains, as above), pass B the levels (certified in fp32,
// the rest listed and resolved after the pass by an 8-way split fp64 sum
// with the reference chain only as the last resort).  The per-tensor scale
// is CTA-local, so there is no grid-wide step; the second read of the
// tensor's 1-2 MB mostly hits L2.  Same warp roles as the one-pass kernel:
// TMA warp, MMA warp (M = 128, N = 3 k, K = d: 2 x 64-column SWIZZLE_128B
// boxes per tile for d = 128), 4 norm warps (the row's |q|), two groups of
// 4 drain warps (tiles g = group mod 2; TMEM slot g & 1).
// The accumulation error dominates the certification margin, so the P1
// part (the leading 8 bits of P, i.e. almost all of x) is accumulated in
// d / 32 separate 32-row chunks (TMEM columns of their own) and summed in
// fp32 after the drain: the worst-case bound of a 32-term accumulation
// replaces that of a d-term one (e = (32 + d/64 + 2) 2^-22 |q| |p_j| +
// 3 2^-24 |x^| instead of d 2^-22 |q| |p_j| + 2^-23 |x^|: ~3.6x tighter at
// d = 128, so ~0.5 % of the 8-bit levels stay uncertified instead of ~1.7 %).
// P2 | P3 (P's bits 9-24, 2^-8 of the magnitude) accumulate over all of d.
template <int D, int KD>
struct Tensor2Smem {
    static constexpr int N = 3 * KD;
    static constexpr int kChunks = D / 32;               // P1 accumulation chunks
    static constexpr int kCols = 2 * KD + kChunks * KD;  // TMEM columns per tile: P2 | P3 | P1 chunks
    static constexpr int kStages = D == 128 ? 3 : 4;
    static constexpr int kTile = 128 * D * 2;
    static constexpr int kList = 4096;         // u32 entries (pass A: (entry, bound) pairs)
    static constexpr int kMaxT2 = 2 * 128;     // ready flags: 2 passes x L <= 16384
    static constexpr int oRing = 0;
    static constexpr int oImg = oRing + kStages * kTile;
    static constexpr int oPn = oImg + N * D * 2;
    static constexpr int oPd = oPn + 256;
    static constexpr int oDq = oPd + D * KD * 8;  // [kStages][128] floats
    static constexpr int oList = oDq + kStages * 128 * 4;
    static constexpr int oBar = oList + kList * 4;
    static constexpr int oMisc = oBar + (2 * kStages + 4) * 8;
    static constexpr int oReady = oMisc + 64;
    static constexpr int bytes = oReady + kMaxT2 * 4;
};

// Level of column j of X row `row` (global), bit-identical to the
// reference's clamp(round_half_away(chain / s)): 8-way split sum of the
// exact fp64 products, certified against the chain's and the sum's error
// bound (as project_tc.cu's level_split); the chain itself only within
// ~1e-14 relative of a .5 boundary.
template <int D, int KD>
__device__ __noinline__ float level_split_g(const __nv_bfloat16* __restrict__ row, const double* pd, int j, double s,
                                            double inv_s, double qmax, int round_f32) {
    if (round_f32)
        return static_cast<float>(fmin(fmax(round_half_away(chain_g<D, KD>(row, pd, j, 1) / s), -qmax), qmax));
    uint4 xr[D / 8];
#pragma unroll
    for (int c = 0; c < D / 8; ++c) xr[c] = __ldg(reinterpret_cast<const uint4*>(row) + c);
    double ps[8], pa[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) ps[u] = pa[u] = 0.0;
#pragma unroll
    for (int c = 0; c < D / 8; ++c) {
        const __nv_bfloat16* xe = reinterpret_cast<const __nv_bfloat16*>(&xr[c]);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double pr = to_double(xe[u]) * pd[(c * 8 + u) * KD + j];
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
    return static_cast<float>(fmin(fmax(round_half_away(chain_g<D, KD>(row, pd, j, 0) / s), -qmax), qmax));
}

template <int D, int KD, bool CH>
__global__ void __launch_bounds__(kThreads, 1)
    project_tensor2_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                           const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                           const float* __restrict__ p, int64_t L, int round_f32, double qmax,
                           uint16_t* __restrict__ lq, uint16_t* __restrict__ lk, double* __restrict__ sq,
                           double* __restrict__ sk) {
    using Sm = Tensor2Smem<D, KD>;
    constexpr int N = Sm::N, S = Sm::kStages, kH = D / 64;
    static_assert(Sm::kCols <= 256, "one 256-column TMEM slot per tile");
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* ring = sm + Sm::oRing;
    unsigned char* img = sm + Sm::oImg;
    float* pn = reinterpret_cast<float*>(sm + Sm::oPn);
    double* pd = reinterpret_cast<double*>(sm + Sm::oPd);
    float* dq_st = reinterpret_cast<float*>(sm + Sm::oDq);
    uint32_t* list = reinterpret_cast<uint32_t*>(sm + Sm::oList);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + Sm::oBar);
    uint64_t* empty = full + S;
    uint64_t* accf = full + 2 * S;  // [2]
    uint64_t* acce = accf + 2;      // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + Sm::oMisc);
    unsigned* lb_u = tslot + 1;
    unsigned* cnt = tslot + 2;  // [2]
    unsigned long long* am_u = reinterpret_cast<unsigned long long*>(sm + Sm::oMisc + 16);
    unsigned* ready = reinterpret_cast<unsigned*>(sm + Sm::oReady);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int which = static_cast<int>(blockIdx.x & 1);
    const int64_t pair = blockIdx.x >> 1;
    const int T = static_cast<int>((L + 127) / 128), TT = 2 * T;
    const __nv_bfloat16* X = (which ? k : q) + pair * L * D;
    const CUtensorMap* map = which ? &mk : &mq;
    auto load_tile = [&](int g) {  // tile g % T of pass g / T
        const int s = g % S, t = g % T;
        tc::mbar_expect_tx(&full[s], Sm::kTile);
#pragma unroll
        for (int h = 0; h < kH; ++h)
            tc::tma_load_2d(tc::smem_addr(ring + s * Sm::kTile + h * (128 * 128)), map, h * 64,
                            static_cast<int>(pair * L + t * 128), &full[s]);
    };
    if (warp == 8 && lane == 0) {
        for (int s2 = 0; s2 < S; ++s2) {
            tc::mbar_init(&full[s2], 1);
            tc::mbar_init(&empty[s2], 1 + 4 + 4);  // MMA commit + the 4 norm warps + the tile's 4 drain warps
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&accf[a], 1);
            tc::mbar_init(&acce[a], 4);
        }
        tc::fence_barrier_init();
        for (int g = 0; g < min(S, TT); ++g) load_tile(g);
    }
    // prologue: P split exactly into three bf16 parts (B-operand image) and
    // P in f64 for the chains
    constexpr int kPer = (D * KD + kThreads - 1) / kThreads;
    float pv[kPer];
#pragma unroll
    for (int m = 0; m < kPer; ++m) pv[m] = tid + m * kThreads < D * KD ? __ldg(p + tid + m * kThreads) : 0.f;
#pragma unroll
    for (int m = 0; m < kPer; ++m) {
        const int i = tid + m * kThreads;
        if (i >= D * KD) break;
        const int c = i / KD, j = i % KD;
        const float v = pv[m];
        pd[i] = static_cast<double>(v);
        const __nv_bfloat16 b1 = __float2bfloat16_rn(v);
        const float r1 = v - __bfloat162float(b1);
        const __nv_bfloat16 b2 = __float2bfloat16_rn(r1);
        const float r2 = r1 - __bfloat162float(b2);
        *reinterpret_cast<__nv_bfloat16*>(img + img_off<D>(j, c)) = b1;
        *reinterpret_cast<__nv_bfloat16*>(img + img_off<D>(KD + j, c)) = b2;
        *reinterpret_cast<__nv_bfloat16*>(img + img_off<D>(2 * KD + j, c)) = __float2bfloat16_rn(r2);
    }
    for (int i = tid; i < TT; i += kThreads) ready[i] = 0u;
    if (tid == 0) {
        *lb_u = 0u;
        cnt[0] = cnt[1] = 0u;
        *am_u = 0ull;
    }
    if (warp == 9) tc::tmem_alloc<512>(tslot);
    tc::fence_proxy_async();  // the P image (generic stores) -> the MMA's async proxy
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tslot;
    // CH: three fp32 roundings combine the partial sums (|x^| 3 2^-24), else
    // two (2^-23); plus the reference's own f32 rounding when it rounds
    // through float
    const float rel = CH ? (round_f32 ? 3.0e-7f : 1.8e-7f) : (round_f32 ? 2.4e-7f : 1.2e-7f);

    if (warp == 8) {
        if (lane == 0)
            for (int g = S; g < TT; ++g) {
                tc::mbar_wait_sleep<64>(&empty[g % S], ((g / S) & 1) ^ 1);
                load_tile(g);
            }
    } else if (warp == 9) {
        if (lane == 0) {
            constexpr uint32_t id23 = tc::idesc_bf16_f32(128, 2 * KD), id1 = tc::idesc_bf16_f32(128, KD);
            const uint32_t bs = tc::smem_addr(img);
            for (int g = 0; g < TT; ++g) {
                const int s = g % S, a = g & 1;
                tc::mbar_wait_sleep<32>(&full[s], (g / S) & 1);
                tc::mbar_wait_sleep<32>(&acce[a], ((g >> 1) & 1) ^ 1);
                tc::fence_after_sync();
                const uint32_t xs = tc::smem_addr(ring + s * Sm::kTile);
                const uint32_t acc = tmem + a * 256;
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint64_t ad = tc::desc_sw128(xs + (ks >> 2) * (128 * 128) + (ks & 3) * 32, 16, 1024);
                    if constexpr (!CH) {  // P1 | P2 | P3 in one accumulation -> columns [0, 3KD)
                        tc::mma_bf16(acc, ad, tc::desc_kmajor_nosw(bs + ks * 256, 128, D * 16),
                                     tc::idesc_bf16_f32(128, 3 * KD), ks > 0);
                        continue;
                    }
                    // P2 | P3 (image rows KD..3KD) over all of d -> columns [0, 2KD)
                    const uint64_t b23 = tc::desc_kmajor_nosw(bs + (KD / 8) * (D * 16) + ks * 256, 128, D * 16);
                    tc::mma_bf16(acc, ad, b23, id23, ks > 0);
                    // P1 (image rows 0..KD) per 32-row chunk of d -> columns 2KD + chunk KD
                    const uint64_t b1 = tc::desc_kmajor_nosw(bs + ks * 256, 128, D * 16);
                    tc::mma_bf16(acc + 2 * KD + (ks >> 1) * KD, ad, b1, id1, ks & 1);
                }
                tc::commit(&accf[a]);
                tc::commit(&empty[s]);
            }
        }
    } else if (warp >= 10) {
        // norm warps: |q| of every row of every tile of both passes
        const int rr = (warp - 10) * 32 + lane;
        for (int g = 0; g < TT; ++g) {
            const int s = g % S;
            tc::mbar_wait_sleep<32>(&full[s], (g / S) & 1);
            const unsigned char* tile = ring + s * Sm::kTile;
            float2 a2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int h = 0; h < kH; ++h)
#pragma unroll
                for (int ch = 0; ch < 8; ++ch) {
                    const uint4 v = *reinterpret_cast<const uint4*>(tile + h * (128 * 128) + rr * 128 + ((ch ^ (rr & 7)) << 4));
                    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float2 f = make_float2(__uint_as_float(wv[u] << 16), __uint_as_float(wv[u] & 0xffff0000u));
                        a2 = __ffma2_rn(f, f, a2);
                    }
                }
            // |q| (32 + d/64 + 2) 2^-22: the chunked accumulation bound (see Tensor2Smem)
            dq_st[s * 128 + rr] = (sqrtf(a2.x + a2.y) * 1.001f + 1e-30f) *
                                  (static_cast<float>(CH ? 32 + D / 64 + 2 : D) * 2.384185791015625e-7f);
            __syncwarp();
            if (lane == 0) {
                tc::mbar_arrive(&empty[s]);
                __threadfence_block();
                atomicAdd(&ready[g], 1u);
            }
        }
    } else {
        // drain groups: group gr takes the tiles g with g & 1 == gr (TMEM slot gr)
        const int gr = warp >> 2, rr = (warp & 3) * 32 + lane;
        const uint32_t lanes = static_cast<uint32_t>((warp & 3) * 32) << 16;
        float pm;  // max_j |p_j| 1.001
        {
            constexpr int kSplit = 32 / KD;  // lanes per column
            const int j = lane % KD, h = lane / KD;
            double s2 = 0.0;
#pragma unroll 8
            for (int u = h * (D / kSplit); u < (h + 1) * (D / kSplit); ++u) s2 = fma(pd[u * KD + j], pd[u * KD + j], s2);
            if (kSplit == 2) s2 += __shfl_xor_sync(0xffffffffu, s2, KD);
            float v = static_cast<float>(sqrt(s2) * 1.001);
            if (warp == 0 && lane < KD) pn[lane] = v;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
            pm = v;
        }
        // one tile: drain x^, the row's dq; frees the TMEM slot and (after dq) the stage
        auto drain = [&](int g, float (&x)[KD], float& dq) {
            const int s = g % S, a = g & 1;
            tc::mbar_wait(&accf[a], (g >> 1) & 1);
            tc::fence_after_sync();
            // x^ = (sum of the P1 chunks, pairwise) + (P2 + P3)
            const uint32_t base = tmem + lanes + a * 256;
            float y[KD];
            if constexpr (!CH) {  // x^ = P1 + (P2 + P3), columns [0, 3KD)
                uint32_t u0[32], u1[32], u2[32];
                if constexpr (KD == 16) {
                    tc::ld_32x32b_x32(base, u0);
                    tc::ld_32x32b_x16(base + 32, *reinterpret_cast<uint32_t(*)[16]>(u1));
                } else {
                    tc::ld_32x32b_x32(base, u0);
                    tc::ld_32x32b_x32(base + 32, u1);
                    tc::ld_32x32b_x32(base + 64, u2);
                }
                tc::wait_ld();
#pragma unroll
                for (int j = 0; j < KD; ++j) {
                    if constexpr (KD == 16)
                        y[j] = __uint_as_float(u0[j]) + (__uint_as_float(u0[16 + j]) + __uint_as_float(u1[j]));
                    else
                        y[j] = __uint_as_float(u0[j]) + (__uint_as_float(u1[j]) + __uint_as_float(u2[j]));
                }
            } else if constexpr (KD == 16) {
                uint32_t u0[32], u1[32];
                tc::ld_32x32b_x32(base, u0);       // P2 | P3
                tc::ld_32x32b_x32(base + 32, u1);  // P1 chunks 0 | 1
                float c23[16];
                if constexpr (D == 128) {
                    uint32_t u2[32];
                    tc::ld_32x32b_x32(base + 64, u2);  // P1 chunks 2 | 3
                    tc::wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; ++j) c23[j] = __uint_as_float(u2[j]) + __uint_as_float(u2[16 + j]);
                } else {
                    tc::wait_ld();
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    float c = __uint_as_float(u1[j]) + __uint_as_float(u1[16 + j]);
                    if constexpr (D == 128) c = c + c23[j];
                    y[j] = c + (__uint_as_float(u0[j]) + __uint_as_float(u0[16 + j]));
                }
            } else {
                uint32_t u0[32], u1[32];
                float c[32];
                tc::ld_32x32b_x32(base + 64, u0);  // P1 chunk 0
                tc::ld_32x32b_x32(base + 96, u1);  // P1 chunk 1
                tc::wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j) c[j] = __uint_as_float(u0[j]) + __uint_as_float(u1[j]);
                if constexpr (D == 128) {
                    tc::ld_32x32b_x32(base + 128, u0);  // P1 chunk 2
                    tc::ld_32x32b_x32(base + 160, u1);  // P1 chunk 3
                    tc::wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) c[j] = c[j] + (__uint_as_float(u0[j]) + __uint_as_float(u1[j]));
                }
                tc::ld_32x32b_x32(base, u0);       // P2
                tc::ld_32x32b_x32(base + 32, u1);  // P3
                tc::wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j) y[j] = c[j] + (__uint_as_float(u0[j]) + __uint_as_float(u1[j]));
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&acce[a]);
#pragma unroll
            for (int j = 0; j < KD; ++j) x[j] = y[j];
            while (*reinterpret_cast<volatile unsigned*>(&ready[g]) < 4u) __nanosleep(32);
            __threadfence_block();
            dq = dq_st[s * 128 + rr];
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&empty[s]);
        };
        // ---- pass A: candidates of the maximum against the running lower bound
        float lb = 0.f;
        for (int g = gr; g < T; g += 2) {
            float xv[KD], dq;
            drain(g, xv, dq);
            float xm = 0.f;
#pragma unroll
            for (int j = 0; j < KD; ++j) xm = fmaxf(xm, fabsf(xv[j]));
            const float er = fmaf(dq, pm, xm * rel) + 1e-30f;
            const int64_t row = static_cast<int64_t>(g) * 128 + rr;
            const bool valid = row < L;
            float lbw = valid ? fmaxf(0.f, (xm - er) * 0.999999f) : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) lbw = fmaxf(lbw, __shfl_xor_sync(0xffffffffu, lbw, o));
            lb = fmaxf(lb, lbw);
            if (lane == 0) atomicMax(lb_u, __float_as_uint(lb));
            const float thr = fmaxf(lb, __uint_as_float(*reinterpret_cast<volatile unsigned*>(lb_u))) - er;
            const bool cand = valid && xm >= thr;
            if (__any_sync(0xffffffffu, cand) && cand) {
#pragma unroll
                for (int j = 0; j < KD; ++j) {
                    const float ax = fabsf(xv[j]);
                    if (ax < thr) continue;
                    const unsigned slot = atomicAdd(&cnt[0], 1u);
                    if (slot < Sm::kList / 2) {
                        list[2 * slot] = (static_cast<uint32_t>(row) << 6) | j;
                        list[2 * slot + 1] = __float_as_uint(ax + er);
                    } else {
                        atomicMax(am_u, static_cast<unsigned long long>(__double_as_longlong(
                                            fabs(chain_g<D, KD>(X + row * D, pd, j, round_f32)))));
                    }
                }
            }
        }
        // ---- the amax: the recorded candidates passing the final bound, one chain each
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
        {
            const unsigned n = min(cnt[0], static_cast<unsigned>(Sm::kList / 2));
            const float LB = __uint_as_float(*lb_u);
            for (unsigned e = tid; e < n; e += 256)
                if (__uint_as_float(list[2 * e + 1]) >= LB)
                    atomicMax(am_u, static_cast<unsigned long long>(__double_as_longlong(fabs(chain_g<D, KD>(
                                        X + static_cast<int64_t>(list[2 * e] >> 6) * D, pd, list[2 * e] & 63, round_f32)))));
        }
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
        const double am = __longlong_as_double(static_cast<long long>(*am_u));
        const double s = am / qmax;
        if (tid == 0) (which ? sk : sq)[pair] = am == 0.0 ? 0.0 : s;
        uint16_t* out = (which ? lk : lq) + pair * L * KD;
        // ---- pass B: levels, certified when |t - rint(t)| + the row's largest margin < 1/2
        const float inv_s = static_cast<float>(qmax / am);
        const float k1 = 1e-6f + 1.001f * rel;
        const float kq = static_cast<float>(qmax + 0.5) * k1;
        const float2 inv2 = make_float2(inv_s, inv_s);
        const float2 mg2 = make_float2(12582912.f, 12582912.f);
        const float2 nmg2 = make_float2(-12582912.f, -12582912.f);
        for (int g = T + ((gr - T) & 1); g < TT; g += 2) {
            float xv[KD], dq;
            drain(g, xv, dq);
            const int64_t row = static_cast<int64_t>(g - T) * 128 + rr;
            if (row >= L) continue;
            const float arow = dq * inv_s * 1.001f;
            uint32_t w[KD / 2];
            float dv[KD];
            float dmax = 0.f;
#pragma unroll
            for (int h = 0; h < KD / 2; ++h) {
                const float2 x2 = make_float2(xv[2 * h], xv[2 * h + 1]);
                const float2 b = __ffma2_rn(x2, inv2, mg2);
                const float2 r = __fadd2_rn(b, nmg2);
                const float2 d = __ffma2_rn(x2, inv2, make_float2(-r.x, -r.y));
                dv[2 * h] = d.x;
                dv[2 * h + 1] = d.y;
                dmax = fmaxf(dmax, fmaxf(fabsf(d.x), fabsf(d.y)));
                const uint32_t lo = __float_as_uint(r.x) | (__float_as_uint(x2.x) & 0x80000000u);
                const uint32_t hi = __float_as_uint(r.y) | (__float_as_uint(x2.y) & 0x80000000u);
                w[h] = __byte_perm(lo, hi, 0x7632);
            }
            if (am == 0.0) {
#pragma unroll
                for (int h = 0; h < KD / 2; ++h) w[h] = 0u;
            }
#pragma unroll
            for (int c = 0; c < KD / 8; ++c)
                *reinterpret_cast<uint4*>(out + lvl_index(L, row, c * 8)) =
                    make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
            const float dthr = 0.5f - fmaf(arow, pm, kq);
            if (dmax >= dthr && am != 0.0) {
                unsigned um = 0;
#pragma unroll
                for (int j = 0; j < KD; ++j) um |= (fabsf(dv[j]) >= dthr ? 1u : 0u) << j;
#pragma unroll 1
                while (um) {
                    const int j = __ffs(um) - 1;
                    um &= um - 1u;
                    const unsigned slot = atomicAdd(&cnt[1], 1u);
                    if (slot < Sm::kList) {
                        list[slot] = (static_cast<uint32_t>(row) << 6) | j;
                    } else {
                        const float lv = level_split_g<D, KD>(X + row * D, pd, j, s, qmax / am, qmax, round_f32);
                        out[lvl_index(L, row, j)] = static_cast<uint16_t>(__float_as_uint(lv) >> 16);
                    }
                }
            }
        }
        // ---- the listed levels (their stored fp32 level is overwritten)
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
        {
            const unsigned n = min(cnt[1], static_cast<unsigned>(Sm::kList));
            const double inv_d = qmax / am;
            for (unsigned e = tid; e < n; e += 256) {
                const int64_t row = static_cast<int64_t>(list[e] >> 6);
                const int j = static_cast<int>(list[e] & 63);
                const float lv = level_split_g<D, KD>(X + row * D, pd, j, s, inv_d, qmax, round_f32);
                out[lvl_index(L, row, j)] = static_cast<uint16_t>(__float_as_uint(lv) >> 16);
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 9) tc::tmem_dealloc<512>(tmem);
}

}  // namespace

bool predict_tensor_supported(const PredictArgs& a) {
    if (!a.bf16 || a.per_row || options().predict_tiles) return false;
    if (a.D != 64 || a.KD != 16 || a.L < 1 || a.L > 128 * TensorSmem<64, 16>::kMaxTiles) return false;
    if (a.pairs < 1 || a.pairs * a.L > INT_MAX || 2 * a.pairs > INT_MAX) return false;
    const auto al = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) == 0; };
    return al(a.q) && al(a.k) && a.lq != nullptr && a.lk != nullptr;
}

void run_predict_tensor(const PredictArgs& a, cudaStream_t st) {
    using Sm = TensorSmem<64, 16>;
    auto kf = project_tensor_kernel<64, 16>;
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, Sm::bytes);
    const CUtensorMap mq = make_map(a.q, a.pairs * a.L, 64, 128, 64);
    const CUtensorMap mk = make_map(a.k, a.pairs * a.L, 64, 128, 64);
    kf<<<static_cast<unsigned>(2 * a.pairs), kThreads, Sm::bytes, st>>>(
        mq, mk, static_cast<const __nv_bfloat16*>(a.q), static_cast<const __nv_bfloat16*>(a.k), a.p, a.L,
        a.round_f32, a.qmax, a.lq, a.lk, a.sq, a.sk);
    note_launch();
}

bool predict_tensor2_supported(const PredictArgs& a) {
    if (!a.bf16 || a.per_row || options().predict_tiles) return false;
    if (!((a.D == 64 && a.KD == 16) || (a.D == 128 && a.KD == 32) || (a.D == 128 && a.KD == 16) || (a.D == 64 && a.KD == 32)))
        return false;
    if (a.L < 1 || a.L > 128 * 128 || a.pairs < 1 || a.pairs * a.L > INT_MAX || 2 * a.pairs > INT_MAX) return false;
    const auto al = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) == 0; };
    return al(a.q) && al(a.k) && a.lq != nullptr && a.lk != nullptr;
}

// chunked P1 accumulation (tighter certification) where levels are fine
// enough for it to matter (> 4 bits); coarse levels take one accumulation
template <int D, int KD>
static void launch_tensor2(const PredictArgs& a, cudaStream_t st) {
    using Sm = Tensor2Smem<D, KD>;
    auto kf = a.qmax > 7.5 ? project_tensor2_kernel<D, KD, true> : project_tensor2_kernel<D, KD, false>;
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, Sm::bytes);
    const CUtensorMap mq = make_map(a.q, a.pairs * a.L, D, 128, 64);
    const CUtensorMap mk = make_map(a.k, a.pairs * a.L, D, 128, 64);
    kf<<<static_cast<unsigned>(2 * a.pairs), kThreads, Sm::bytes, st>>>(
        mq, mk, static_cast<const __nv_bfloat16*>(a.q), static_cast<const __nv_bfloat16*>(a.k), a.p, a.L,
        a.round_f32, a.qmax, a.lq, a.lk, a.sq, a.sk);
    note_launch();
}

void run_predict_tensor2(const PredictArgs& a, cudaStream_t st) {
    if (a.D == 64) {
        if (a.KD == 16) launch_tensor2<64, 16>(a, st);
        else launch_tensor2<64, 32>(a, st);
    } else {
        if (a.KD == 16) launch_tensor2<128, 16>(a, st);
        else launch_tensor2<128, 32>(a, st);
    }
}

}  // namespace dsa

#ifdef DSA_PT_PROBE
extern "C" int dsa_pt_count_read(unsigned* out, int n) {
    return static_cast<int>(cudaMemcpyFromSymbol(out, dsa::g_pt_count, sizeof(unsigned) * 2 * n));
}
extern "C" int dsa_pt_probe_read(unsigned long long* out, int n) {
    return static_cast<int>(cudaMemcpyFromSymbol(out, dsa::g_pt_probe, sizeof(unsigned long long) * 8 * n));
}
#endif
