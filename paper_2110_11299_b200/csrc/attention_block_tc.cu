// Phase 3 for block masks (C3: 32 x 32 blocks, d = 128) on the 5th-gen
// tensor cores: every kept block's K and V rows arrive by TMA, both GEMMs run
// as tcgen05.mma with the accumulators in TMEM.
//
// Reference: sddmm -> sparse_softmax -> spmm per head (P/src/sparse.cpp:38-91)
// over the block mask (block row ib keeps `keep` blocks of 32 keys):
// per query row, s_j = <q_i, k_j> / sqrt(d) over the kept keys, a softmax, and
// z_i = sum_j p_j v_j.
//
// One CTA = one block row (32 queries) of one (b,h) pair; its kept keys are
// `keep` blocks x 32 = up to 512 keys, taken in groups of 4 blocks (128 keys):
//
//   S^T[key, q] = K_group . Q^T      tcgen05.mma kind::f16, M = 128 keys,
//                                     N = 32 queries, K = d; A and B K-major,
//                                     128-byte-swizzled TMA tiles; each group's
//                                     32 fp32 columns stay in TMEM (<= 128)
//   softmax over the keys of every query column, EXACT (no online
//   rescaling): thread = TMEM lane = key; the column maxima and sums are
//   warp transpose-reductions (31 shuffles) plus a 4-warp combine in shared
//   memory; P^T (bf16) is written MN-major, 16 bytes per (key, 8 queries)
//   Z^T[d, q] = V^T . P^T             tcgen05.mma, M = d = 128, N = 32, K =
//                                     the keys; A = the V rows as TMA loaded
//                                     them (MN-major, 128-byte swizzle), B =
//                                     P^T (MN-major, no swizzle)
//   thread = TMEM lane = d: z / l per query column, stored as Z rows.
//
// A producer lane streams the 8 operand groups (K0..K3 then V0..V3) through a
// two-stage ring (4 blocks x 2 d-halves = 8 TMA boxes of 32 x 64 per group);
// the V loads overlap the softmax.  Every kept block's K and V rows cross
// L2 -> SM once per block row (the compulsory gather of this mask).
#include <cuda.h>
#include <cuda_bf16.h>

#include "device_common.cuh"
#include "kernels.h"
#include "tc_sm100.cuh"
#include "tma_map.h"

namespace dsa {
namespace {

constexpr int kD = 128;             // head width
constexpr int kBlk = 32;            // block edge
constexpr int kG = 4;               // blocks per key group (M = 128 keys)
constexpr int kMaxGroups = 4;       // keep <= 16 blocks (S^T in <= 128 TMEM columns)
constexpr int kHalf = kG * kBlk * 128;       // one d-half (64 columns) of a group: 16 KB
constexpr int kStage = 2 * kHalf;            // K or V group: 32 KB
constexpr int kQBytes = kBlk * kD * 2;       // 8 KB (two 4 KB d-halves)
constexpr int kPBytes = kMaxGroups * kG * kBlk * kBlk * 2;  // P^T: 512 keys x 32 q, 32 KB
constexpr int kEpi = 4;                      // softmax / output warps (128 TMEM lanes)
constexpr int kThreads = (kEpi + 1) * 32;
constexpr int kSmem = 1024 + 2 * kStage + kQBytes + kPBytes + 2 * 4 * 32 * 4 + 256;

__device__ __forceinline__ float bc_ex2(float x) {  // 2^x on the SFU
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(kEpi * 32) : "memory"); }

// transpose-reduction over a warp: lane l ends with the reduction of
// column l over the warp's 32 lanes (31 shuffles)
template <bool MAX>
__device__ __forceinline__ float warp_colreduce(float (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            // keep half [up ? o : 0, +o), send the other half
            const float mine = up ? v[i + o] : v[i];
            const float other = up ? v[i] : v[i + o];
            const float got = __shfl_xor_sync(0xffffffffu, other, o);
            v[i] = MAX ? fmaxf(mine, got) : mine + got;
        }
    }
    return v[0];
}

__global__ void __launch_bounds__(kThreads, 2)
    attn_block_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                         const __grid_constant__ CUtensorMap map_v, const uint32_t* __restrict__ block_cols,
                         int L, int keep, int scale, __nv_bfloat16* __restrict__ Z) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
    unsigned char* stage_p = smem;                       // [2][kStage], 1024-aligned
    unsigned char* q_p = stage_p + 2 * kStage;           // [2 halves][32 rows][128 B]
    unsigned char* p_p = q_p + kQBytes;                  // P^T, MN-major, no swizzle
    float* red = reinterpret_cast<float*>(p_p + kPBytes);  // [4 warps][32] partials
    float* colv = red + 4 * 32;                          // [32] column max, then 1/sum
    uint64_t* bars = reinterpret_cast<uint64_t*>(colv + 32 + 32);
    uint64_t* full = bars;       // [2]
    uint64_t* empty = bars + 2;  // [2]
    uint64_t* qbar = bars + 4;
    uint64_t* sbar = bars + 5;   // S^T complete
    uint64_t* pbar = bars + 6;   // P^T written
    uint64_t* zbar = bars + 7;   // Z^T complete
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t pair = blockIdx.y;
    const int ib = blockIdx.x;
    const int nbr = L / kBlk;
    const uint32_t* blist = block_cols + (pair * nbr + ib) * static_cast<int64_t>(keep);
    const int ng = (keep + kG - 1) / kG;
    const int row_q = static_cast<int>(pair * L) + ib * kBlk;  // Q / Z row of query 0

    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 1);
        }
        tc::mbar_init(qbar, 1);
        tc::mbar_init(sbar, 1);
        tc::mbar_init(pbar, 1);
        tc::mbar_init(zbar, 1);
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<256>(tmem_slot);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;  // S^T: columns [0, 32 ng); Z^T: [128, 160)

    if (warp == kEpi) {
        // ---------------------------------------- TMA producer + MMA issuer
        if (lane == 0) {
            const uint32_t st0 = tc::smem_addr(stage_p), q_s = tc::smem_addr(q_p), p_s = tc::smem_addr(p_p);
            tc::mbar_expect_tx(qbar, kQBytes);
            tc::tma_load_2d(q_s, &map_q, 0, row_q, qbar);
            tc::tma_load_2d(q_s + kQBytes / 2, &map_q, 64, row_q, qbar);
            // load li: groups 0..ng-1 of K, then of V; a missing block of the
            // last group repeats a kept one (finite data, masked / P = 0)
            auto load = [&](int li) {
                const int s = li & 1;
                const bool isv = li >= ng;
                const int g = isv ? li - ng : li;
                if (li >= 2) tc::mbar_wait_sleep(&empty[s], ((li >> 1) - 1) & 1);
                tc::mbar_expect_tx(&full[s], kStage);
                const uint32_t dst = st0 + s * kStage;
#pragma unroll
                for (int b = 0; b < kG; ++b) {
                    const int slot = g * kG + b;
                    const int blk = static_cast<int>(__ldg(blist + (slot < keep ? slot : keep - 1)));
                    const int row = static_cast<int>(pair * L) + blk * kBlk;
                    const CUtensorMap* m = isv ? &map_v : &map_k;
                    tc::tma_load_2d(dst + b * (kBlk * 128), m, 0, row, &full[s]);
                    tc::tma_load_2d(dst + kHalf + b * (kBlk * 128), m, 64, row, &full[s]);
                }
            };
            const int nload = 2 * ng;
            int next = 0;
            for (; next < 2 && next < nload; ++next) load(next);
            // S^T = K_group . Q^T: M = 128 keys, N = 32, K = 128 (two 64-wide halves)
            const uint32_t id1 = tc::idesc_bf16_f32(128, kBlk);
            tc::mbar_wait(qbar, 0);
            for (int g = 0; g < ng; ++g) {
                const int s = g & 1;
                tc::mbar_wait(&full[s], (g >> 1) & 1);
                tc::fence_after_sync();
#pragma unroll
                for (int ks = 0; ks < kD / 16; ++ks) {
                    const int h = ks >> 2, kk = ks & 3;  // d-half, 16-column step inside it (32 B)
                    const uint64_t ad = tc::desc_sw128(st0 + s * kStage + h * kHalf + kk * 32, 16, 1024);
                    const uint64_t bd = tc::desc_sw128(q_s + h * (kQBytes / 2) + kk * 32, 16, 1024);
                    tc::mma_bf16(tmem + g * kBlk, ad, bd, id1, ks > 0);
                }
                tc::commit(&empty[s]);
                if (next < nload) load(next++);
            }
            tc::commit(sbar);
            // Z^T = V^T . P^T: M = d = 128, N = 32, K = the keys; A = V (MN-major,
            // swizzled: d-halves 16 KB apart (LBO), 8-key atoms 1024 B (SBO)),
            // B = P^T (MN-major, no swizzle: 8-query chunks 128 B apart (SBO),
            // 8-key groups 512 B (LBO))
            const uint32_t id2 = tc::idesc_bf16_f32_mn(128, kBlk, true, true);
            tc::mbar_wait_sleep(pbar, 0);
            tc::fence_after_sync();
            for (int g = 0; g < ng; ++g) {
                const int li = ng + g, s = li & 1;
                tc::mbar_wait(&full[s], (li >> 1) & 1);
                tc::fence_after_sync();
#pragma unroll
                for (int kk = 0; kk < kG * kBlk / 16; ++kk) {
                    const uint64_t ad = tc::desc_sw128(st0 + s * kStage + kk * 2048, kHalf, 1024);
                    const uint64_t bd = tc::desc_kmajor_nosw(p_s + (g * 16 + kk * 2) * 512, 512, 128);
                    tc::mma_bf16(tmem + 128, ad, bd, id2, (g > 0 || kk > 0) ? 1u : 0u);
                }
                tc::commit(&empty[s]);
                if (next < nload) load(next++);
            }
            tc::commit(zbar);
        }
        return;
    }

    // ------------------------------------------------ softmax (thread = key)
    const float c2 = (scale ? rsqrtf(static_cast<float>(kD)) : 1.f) * 1.4426950408889634f;
    const uint32_t tl = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    tc::mbar_wait_susp(sbar, 0);
    tc::fence_after_sync();
    float v[32];
    float acc[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = -INFINITY;
    for (int g = 0; g < ng; ++g) {
        uint32_t r[32];
        tc::ld_32x32b_x32(tl + g * kBlk, r);
        tc::wait_ld();
        const bool kv = g * kG + warp < keep;  // key slot g*4 + warp of this block row
        if (kv) {
#pragma unroll
            for (int q = 0; q < 32; ++q) acc[q] = fmaxf(acc[q], __uint_as_float(r[q]));
        }
    }
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = acc[q];
    red[warp * 32 + lane] = warp_colreduce<true>(v, lane);
    epi_sync();
    if (warp == 0) {
        const float m = fmaxf(fmaxf(red[lane], red[32 + lane]), fmaxf(red[64 + lane], red[96 + lane]));
        colv[lane] = m * c2;
    }
    epi_sync();
    float mc[32];
#pragma unroll
    for (int q = 0; q < 32; q += 4) {
        const float4 x = *reinterpret_cast<const float4*>(&colv[q]);
        mc[q] = x.x;
        mc[q + 1] = x.y;
        mc[q + 2] = x.z;
        mc[q + 3] = x.w;
    }
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = 0.f;
    for (int g = 0; g < ng; ++g) {
        uint32_t r[32];
        tc::ld_32x32b_x32(tl + g * kBlk, r);
        tc::wait_ld();
        const bool kv = g * kG + warp < keep;
        uint32_t pk[16];
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
            const float p0 = kv ? bc_ex2(fmaf(__uint_as_float(r[q]), c2, -mc[q])) : 0.f;
            const float p1 = kv ? bc_ex2(fmaf(__uint_as_float(r[q + 1]), c2, -mc[q + 1])) : 0.f;
            acc[q] += p0;
            acc[q + 1] += p1;
            __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
            pk[q >> 1] = *reinterpret_cast<uint32_t*>(&h);
        }
        // P^T row `key` (MN-major core matrices: 8 keys x 8 queries, 128 B)
        const int key = g * (kG * kBlk) + warp * 32 + lane;
        unsigned char* dst = p_p + (key >> 3) * 512 + (key & 7) * 16;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            *reinterpret_cast<uint4*>(dst + c * 128) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
    }
    tc::fence_proxy_async();  // P^T (generic stores) -> visible to the tensor core
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = acc[q];
    red[warp * 32 + lane] = warp_colreduce<false>(v, lane);
    epi_sync();
    if (tid == 0) tc::mbar_arrive(pbar);
    if (warp == 0) {
        const float l = red[lane] + red[32 + lane] + red[64 + lane] + red[96 + lane];
        colv[lane] = l > 0.f ? 1.f / l : 0.f;
    }
    epi_sync();

    // ------------------------------------------------ output (thread = d)
    tc::mbar_wait_susp(zbar, 0);
    tc::fence_after_sync();
    uint32_t zr[32];
    tc::ld_32x32b_x32(tl + 128, zr);
    tc::wait_ld();
    const int d = warp * 32 + lane;
#pragma unroll
    for (int q = 0; q < 32; ++q)
        Z[static_cast<int64_t>(row_q + q) * kD + d] = __float2bfloat16_rn(__uint_as_float(zr[q]) * colv[q]);
    tc::fence_before_sync();
    epi_sync();
    if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

}  // namespace

bool block_tc_supported(const AttnArgs& a) {
    return a.mode == kBlock && a.bf16 && a.D == kD && a.block == kBlk && a.L % kBlk == 0 && a.keep >= 1 &&
           a.keep <= kG * kMaxGroups && !options().attn_generic;
}

void run_block_tc(const AttnArgs& a, cudaStream_t st) {
    const int64_t rows = a.pairs * a.L;
    const CUtensorMap mq = make_map(a.q, rows, kD, kBlk, 64);
    const CUtensorMap mk = make_map(a.k, rows, kD, kBlk, 64);
    const CUtensorMap mv = make_map(a.v, rows, kD, kBlk, 64);
    cudaFuncSetAttribute(attn_block_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    const dim3 grid(static_cast<unsigned>(a.L / kBlk), static_cast<unsigned>(a.pairs));
    attn_block_tc_kernel<<<grid, kThreads, kSmem, st>>>(mq, mk, mv, a.cols, static_cast<int>(a.L),
                                                         static_cast<int>(a.keep), a.scale,
                                                         static_cast<__nv_bfloat16*>(a.z));
    note_launch();
}

}  // namespace dsa
