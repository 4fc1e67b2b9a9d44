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

#include <algorithm>

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
constexpr int kNS = 4;                       // operand ring stages
constexpr int kQBytes = kBlk * kD * 2;       // 8 KB (two 4 KB d-halves)
constexpr int kPBytes = kMaxGroups * kG * kBlk * kBlk * 2;  // P^T: 512 keys x 32 q, 32 KB
constexpr int kEpi = 8;                      // softmax / output warps: 2 groups x 4 (128 TMEM lanes)
constexpr int kLoadWarp = kEpi, kMmaWarp = kEpi + 1;
constexpr int kThreads = (kEpi + 2) * 32;
constexpr int kSmem = 1024 + kNS * kStage + 2 * kQBytes + 2 * kPBytes + 2 * (4 * 32 + 2 * 32) * 4 + 512;
// TMEM columns: S^T slots [0, 128), [128, 256); Z^T slots [256, 288), [288, 320)
constexpr uint32_t kTmemZ = 256;

__device__ __forceinline__ float bc_ex2(float x) {  // 2^x on the SFU
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// named barriers: 1 + group for one softmax group (4 warps), 3 for all 8 warps
__device__ __forceinline__ void grp_sync(int grp) { asm volatile("bar.sync %0, 128;\n" ::"r"(1 + grp) : "memory"); }
__device__ __forceinline__ void epi_sync_all() { asm volatile("bar.sync 3, %0;\n" ::"n"(kEpi * 32) : "memory"); }

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

// The work list: block rows r = blockIdx.x + j * gridDim.x (j < n) of all
// pairs.  Operand groups are loaded and consumed in ONE order, the MMA
// issuer's: K(0), K(1), V(0), K(2), V(1), ..., K(n-1), V(n-2), V(n-1) --
// S^T(j + 1) is computed while the softmax of row j runs.
struct Item {
    int j;
    bool v;
};
__device__ __forceinline__ Item item_at(int i, int n) {
    if (i == 0) return {0, false};
    if (i >= 2 * n - 1) return {n - 1, true};
    return (i & 1) ? Item{(i + 1) / 2, false} : Item{i / 2 - 1, true};
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_block_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                         const __grid_constant__ CUtensorMap map_v, const uint32_t* __restrict__ block_cols,
                         int L, int64_t nrows, int keep, int scale, __nv_bfloat16* __restrict__ Z) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
    unsigned char* stage_p = smem;                       // [kNS][kStage], 1024-aligned
    unsigned char* q_p = stage_p + kNS * kStage;         // [2 slots][2 halves][32 rows][128 B]
    unsigned char* p_p = q_p + 2 * kQBytes;              // [2 slots] P^T, MN-major, no swizzle
    float* redb = reinterpret_cast<float*>(p_p + 2 * kPBytes);  // per group: [4 warps][32] partials,
                                                                // [32] scaled column max, [32] 1 / column sum
    uint64_t* bars = reinterpret_cast<uint64_t*>(redb + 2 * (4 * 32 + 2 * 32));
    uint64_t* full = bars;                  // [kNS]
    uint64_t* empty = full + kNS;           // [kNS]
    uint64_t* qfull = empty + kNS;          // [2]
    uint64_t* qempty = qfull + 2;           // [2]
    uint64_t* sfull = qempty + 2;           // [2]
    uint64_t* sempty = sfull + 2;           // [2]
    uint64_t* zfull = sempty + 2;           // [2]
    uint64_t* zempty = zfull + 2;           // [2]
    uint64_t* pfull = zempty + 2;           // [2]
    uint64_t* pempty = pfull + 2;           // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nbr = L / kBlk;
    const int n = nrows > blockIdx.x ? static_cast<int>((nrows - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
    const int ng = (keep + kG - 1) / kG;
    auto row_of = [&](int j) -> int64_t { return blockIdx.x + static_cast<int64_t>(j) * gridDim.x; };

    if (tid == 0) {
        for (int i = 0; i < kNS; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&qfull[i], 1);
            tc::mbar_init(&qempty[i], 1);
            tc::mbar_init(&sfull[i], 1);
            tc::mbar_init(&sempty[i], 1);
            tc::mbar_init(&zfull[i], 1);
            tc::mbar_init(&zempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&pfull[i], 1);
            tc::mbar_init(&pempty[i], 1);
        }
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<512>(tmem_slot);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t st0 = tc::smem_addr(stage_p), q_s = tc::smem_addr(q_p), p_s = tc::smem_addr(p_p);

    if (warp == kLoadWarp) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0) {
            int sc = 0;  // operand groups issued
            for (int i = 0; i < 2 * n; ++i) {
                const Item it = item_at(i, n);
                const int64_t r = row_of(it.j);
                const int64_t pair = r / nbr;
                const int ib = static_cast<int>(r % nbr);
                const int row0 = static_cast<int>(pair * L);
                if (!it.v) {
                    const int qs = it.j & 1;
                    if (it.j >= 2) tc::mbar_wait_sleep(&qempty[qs], ((it.j >> 1) - 1) & 1);
                    tc::mbar_expect_tx(&qfull[qs], kQBytes);
                    tc::tma_load_2d(q_s + qs * kQBytes, &map_q, 0, row0 + ib * kBlk, &qfull[qs]);
                    tc::tma_load_2d(q_s + qs * kQBytes + kQBytes / 2, &map_q, 64, row0 + ib * kBlk, &qfull[qs]);
                }
                const uint32_t* blist = block_cols + r * keep;
                const CUtensorMap* m = it.v ? &map_v : &map_k;
                for (int g = 0; g < ng; ++g, ++sc) {
                    const int s = sc % kNS;
                    if (sc >= kNS) tc::mbar_wait_sleep(&empty[s], ((sc / kNS) - 1) & 1);
                    tc::mbar_expect_tx(&full[s], kStage);
                    const uint32_t dst = st0 + s * kStage;
#pragma unroll
                    for (int b = 0; b < kG; ++b) {
                        // a missing block of the last group repeats a kept one
                        // (finite data; masked in S^T, P = 0 in Z^T)
                        const int slot = g * kG + b;
                        const int blk = static_cast<int>(__ldg(blist + (slot < keep ? slot : keep - 1)));
                        tc::tma_load_2d(dst + b * (kBlk * 128), m, 0, row0 + blk * kBlk, &full[s]);
                        tc::tma_load_2d(dst + kHalf + b * (kBlk * 128), m, 64, row0 + blk * kBlk, &full[s]);
                    }
                }
            }
        }
        return;
    }
    if (warp == kMmaWarp) {
        // ------------------------------------------------------- MMA issuer
        if (lane == 0) {
            // S^T = K_group . Q^T: M = 128 keys, N = 32, K = 128 (two 64-wide,
            // 128-byte-swizzled halves; 16-column steps advance 32 B)
            const uint32_t id1 = tc::idesc_bf16_f32(128, kBlk);
            // Z^T = V^T . P^T: M = d = 128, N = 32, K = keys; A = V as loaded
            // (MN-major, swizzled: d-halves 16 KB apart (LBO), 8-key atoms
            // 1024 B (SBO)); B = P^T (MN-major, no swizzle: 8-query chunks
            // 128 B apart (SBO), 8-key groups 512 B (LBO))
            const uint32_t id2 = tc::idesc_bf16_f32_mn(128, kBlk, true, true);
            int sc = 0;
            for (int i = 0; i < 2 * n; ++i) {
                const Item it = item_at(i, n);
                const int sl = it.j & 1;
                if (!it.v) {
                    tc::mbar_wait(&qfull[sl], (it.j >> 1) & 1);
                    if (it.j >= 2) tc::mbar_wait(&sempty[sl], ((it.j >> 1) - 1) & 1);
                } else {
                    tc::mbar_wait(&pfull[sl], (it.j >> 1) & 1);
                    if (it.j >= 2) tc::mbar_wait(&zempty[sl], ((it.j >> 1) - 1) & 1);
                }
                tc::fence_after_sync();
                for (int g = 0; g < ng; ++g, ++sc) {
                    const int s = sc % kNS;
                    tc::mbar_wait(&full[s], (sc / kNS) & 1);
                    tc::fence_after_sync();
                    const uint32_t sb = st0 + s * kStage;
                    if (!it.v) {
#pragma unroll
                        for (int ks = 0; ks < kD / 16; ++ks) {
                            const int h = ks >> 2, kk = ks & 3;
                            const uint64_t ad = tc::desc_sw128(sb + h * kHalf + kk * 32, 16, 1024);
                            const uint64_t bd = tc::desc_sw128(q_s + sl * kQBytes + h * (kQBytes / 2) + kk * 32, 16, 1024);
                            tc::mma_bf16(tmem + sl * 128 + g * kBlk, ad, bd, id1, ks > 0);
                        }
                    } else {
#pragma unroll
                        for (int kk = 0; kk < kG * kBlk / 16; ++kk) {
                            const uint64_t ad = tc::desc_sw128(sb + kk * 2048, kHalf, 1024);
                            const uint64_t bd = tc::desc_kmajor_nosw(p_s + sl * kPBytes + (g * 16 + kk * 2) * 512, 512, 128);
                            tc::mma_bf16(tmem + kTmemZ + sl * kBlk, ad, bd, id2, (g > 0 || kk > 0) ? 1u : 0u);
                        }
                    }
                    tc::commit(&empty[s]);
                }
                if (!it.v) {
                    tc::commit(&sfull[sl]);
                    tc::commit(&qempty[sl]);
                } else {
                    tc::commit(&zfull[sl]);
                    tc::commit(&pempty[sl]);
                }
            }
        }
        return;
    }

    // ------------------ softmax + output: group grp = rows j = grp (mod 2)
    // (their S^T / P^T / Z^T slot is grp); 4 warps = the 128 TMEM lanes
    const float c2 = (scale ? rsqrtf(static_cast<float>(kD)) : 1.f) * 1.4426950408889634f;
    const int grp = warp >> 2, wq = warp & 3, gt = tid & 127;
    const uint32_t tl = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    float* red = redb + grp * (4 * 32 + 2 * 32);
    float* mcv = red + 4 * 32;
    float* linv = mcv + 32;

    // Z rows of row j: thread = TMEM lane = d; columns = the 32 queries
    auto output = [&](int j) {
        const int sl = j & 1;
        tc::mbar_wait_susp(&zfull[sl], (j >> 1) & 1);
        tc::fence_after_sync();
        uint32_t zr[32];
        tc::ld_32x32b_x32(tl + kTmemZ + sl * kBlk, zr);
        tc::wait_ld();
        tc::fence_before_sync();
        const int64_t r = row_of(j);
        const int64_t q0 = (r / nbr) * L + (r % nbr) * kBlk;
        const int d = wq * 32 + lane;
#pragma unroll
        for (int q = 0; q < 32; ++q)
            Z[(q0 + q) * kD + d] = __float2bfloat16_rn(__uint_as_float(zr[q]) * linv[q]);
        grp_sync(grp);
        if (gt == 0) tc::mbar_arrive(&zempty[sl]);
    };

    for (int j = grp; j < n; j += 2) {
        const int sl = grp;
        tc::mbar_wait_susp(&sfull[sl], (j >> 1) & 1);
        tc::fence_after_sync();
        const uint32_t ts = tl + sl * 128;
        float v[32], acc[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[q] = -INFINITY;
        for (int g = 0; g < ng; ++g) {
            if (g * kG + wq >= keep) continue;  // key slot g*4 + wq not kept
            uint32_t r[32];
            tc::ld_32x32b_x32(ts + g * kBlk, r);
            tc::wait_ld();
#pragma unroll
            for (int q = 0; q < 32; ++q) acc[q] = fmaxf(acc[q], __uint_as_float(r[q]));
        }
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = acc[q];
        red[wq * 32 + lane] = warp_colreduce<true>(v, lane);
        grp_sync(grp);
        if (wq == 0)
            mcv[lane] = fmaxf(fmaxf(red[lane], red[32 + lane]), fmaxf(red[64 + lane], red[96 + lane])) * c2;
        grp_sync(grp);
        float mc[32];
#pragma unroll
        for (int q = 0; q < 32; q += 4) {
            const float4 x = *reinterpret_cast<const float4*>(&mcv[q]);
            mc[q] = x.x;
            mc[q + 1] = x.y;
            mc[q + 2] = x.z;
            mc[q + 3] = x.w;
        }
        if (j >= 2) tc::mbar_wait_susp(&pempty[sl], ((j >> 1) - 1) & 1);  // Z^T(j - 2) has read P^T slot
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[q] = 0.f;
        for (int g = 0; g < ng; ++g) {
            const bool kv = g * kG + wq < keep;
            uint32_t r[32];
            tc::ld_32x32b_x32(ts + g * kBlk, r);
            tc::wait_ld();
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
            const int key = g * (kG * kBlk) + wq * 32 + lane;
            unsigned char* dst = p_p + sl * kPBytes + (key >> 3) * 512 + (key & 7) * 16;
#pragma unroll
            for (int c = 0; c < 4; ++c)
                *reinterpret_cast<uint4*>(dst + c * 128) =
                    make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        }
        tc::fence_proxy_async();  // P^T (generic stores) -> visible to the tensor core
        tc::fence_before_sync();
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = acc[q];
        if (j >= 2) output(j - 2);  // the group's previous row (reads linv before it is rewritten)
        red[wq * 32 + lane] = warp_colreduce<false>(v, lane);
        grp_sync(grp);
        if (gt == 0) {
            tc::mbar_arrive(&pfull[sl]);
            tc::mbar_arrive(&sempty[sl]);
        }
        if (wq == 0) {
            const float l = red[lane] + red[32 + lane] + red[64 + lane] + red[96 + lane];
            linv[lane] = l > 0.f ? 1.f / l : 0.f;
        }
        grp_sync(grp);
    }
    {
        const int last = n - 1 - ((n - 1 - grp) & 1);  // this group's last row
        if (last >= grp && last >= 0) output(last);
    }
    tc::fence_before_sync();
    epi_sync_all();
    if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace

bool block_tc_supported(const AttnArgs& a) {
    return a.mode == kBlock && a.bf16 && a.D == kD && a.block == kBlk && a.L % kBlk == 0 && a.keep >= 1 &&
           a.keep <= kG * kMaxGroups && !options().attn_generic && options().block_tc;
}

void run_block_tc(const AttnArgs& a, cudaStream_t st) {
    const int64_t rows = a.pairs * a.L;
    const CUtensorMap mq = make_map(a.q, rows, kD, kBlk, 64);
    const CUtensorMap mk = make_map(a.k, rows, kD, kBlk, 64);
    const CUtensorMap mv = make_map(a.v, rows, kD, kBlk, 64);
    cudaFuncSetAttribute(attn_block_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    const int64_t nrows = a.pairs * (a.L / kBlk);  // block rows of every pair
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(nrows, sm_count()));
    attn_block_tc_kernel<<<grid, kThreads, kSmem, st>>>(mq, mk, mv, a.cols, static_cast<int>(a.L), nrows,
                                                         static_cast<int>(a.keep), a.scale,
                                                         static_cast<__nv_bfloat16*>(a.z));
    note_launch();
}

}  // namespace dsa
