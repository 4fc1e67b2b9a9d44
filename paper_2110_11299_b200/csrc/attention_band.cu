// Phase 3 for vector-wise (COLVEC) masks: every band of 8 query rows shares
// one ascending list of `keep` key columns (P/src/maskgen.cpp:51-59), so the
// band is an 8-wide tensor-core tile.  Per band (one warp):
//
//   S^T[key, q] = K_sel . Q_band^T      mma m16n8k16 (M = 16 gathered keys,
//                                        N = the band's 8 queries, K = d)
//   online softmax over keys per query column (running max / sum in fp32)
//   Z^T[d, q]  += V_sel^T . P^T         mma m16n8k16 (M = d, K = keys)
//
// K/V rows of the band's keys are gathered in chunks with 16-byte cp.async
// into XOR-swizzled shared memory (conflict-free ldmatrix), double-buffered
// so the next chunk's gather overlaps this chunk's math.  The gather is the
// roofline of this phase (each kept key row is fetched once per band, i.e.
// reused by the band's 8 queries -- SURVEY H6); HBM sees Q, K, V, Z once.
#include <cuda_bf16.h>


#include "device_common.cuh"
#include "kernels.h"
#include "band_core.cuh"
#include "tc_sm100.cuh"
#include "tma_map.h"

#ifndef BLK_STAGES  // 2: more CTAs per SM beat a deeper ring (3 stages: 0.67 ms, 4: 0.86 ms on C3)
#define BLK_STAGES 2
#endif

namespace dsa {
namespace {

using namespace bc;


// Same block-row computation with each warp owning NT bands (8 * NT query
// rows, one MMA n-tile each): the K and V fragments a warp loads from shared
// memory (ldmatrix) serve all its n-tiles, so the L1 / shared-memory
// wavefronts per block drop by NT while the CTA (32 / (8 NT) warps) still
// stages every kept block once.
template <int D, int NT>
struct BlockSmemN {
    static constexpr int kWarps = 4 / NT;
    __nv_bfloat16 k[2][32 * D];
    __nv_bfloat16 v[2][32 * D];
    __nv_bfloat16 q[kWarps][NT][8 * D];   // per warp: Q bands, reused to stage Z
    __nv_bfloat16 p[kWarps][NT][8 * 40];  // per warp: [query][key], padded rows
};

template <int D, int NT>
__global__ void __launch_bounds__(128 / NT)
    attn_block_nt_kernel(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K,
                         const __nv_bfloat16* __restrict__ V, const uint32_t* __restrict__ block_cols,
                         int64_t L, int64_t keep, int scale, __nv_bfloat16* __restrict__ Z) {
    constexpr int CHUNK = 32;
    constexpr int kT = 128 / NT;  // threads per CTA
    extern __shared__ __align__(128) unsigned char dsm[];
    using SM = BlockSmemN<D, NT>;
    SM& sm = *reinterpret_cast<SM*>(dsm);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nbr = L / 32;
    const int64_t pair = blockIdx.y, br = blockIdx.x;
    const int64_t r0 = br * 32 + warp * 8 * NT;  // this warp's first row
    const __nv_bfloat16* Kp = K + pair * L * D;
    const __nv_bfloat16* Vp = V + pair * L * D;
    const uint32_t* cols = block_cols + (pair * nbr + br) * keep;
    const int g = lane >> 2, c4 = lane & 3;
    constexpr int kChunks16 = D / 8;

    for (int t = lane; t < NT * 8 * kChunks16; t += 32) {
        const int n = t / (8 * kChunks16), rc = t % (8 * kChunks16);
        const int r = rc / kChunks16, c = rc % kChunks16;
        cp_async16(smem_u32(sm.q[warp][n]) + swz<D>(r, c), Q + (pair * L + r0 + n * 8 + r) * D + c * 8, true);
    }
    // thread owns 16-byte column chunk c of rows rl, rl + RPS, .. of the block
    // (kT is a multiple of the chunks per row, so c is fixed per thread)
    auto load_block = [&](int buf, int ch) {
        static_assert(kT % kChunks16 == 0, "column chunk fixed per thread");
        constexpr int RPS = kT / kChunks16;  // rows per step
        const int c = tid % kChunks16, rl = tid / kChunks16;
        const size_t j0 = static_cast<size_t>(__ldg(cols + ch)) * 32;
        const uint32_t kbs = smem_u32(sm.k[buf]), vbs = smem_u32(sm.v[buf]);
#pragma unroll
        for (int i = 0; i < CHUNK / RPS; ++i) {
            const int r = rl + i * RPS;
            cp_async16(kbs + swz<D>(r, c), Kp + (j0 + r) * D + c * 8, true);
            cp_async16(vbs + swz<D>(r, c), Vp + (j0 + r) * D + c * 8, true);
        }
    };
    const int nchunks = static_cast<int>(keep);
    load_block(0, 0);
    cp_async_commit();

    const float sl2 = (scale ? rsqrtf(static_cast<float>(D)) : 1.f) * 1.4426950408889634f;
    float m_run[NT][2], l_part[NT][2];
    float zacc[NT][D / 16][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        m_run[n][0] = m_run[n][1] = -INFINITY;
        l_part[n][0] = l_part[n][1] = 0.f;
#pragma unroll
        for (int t = 0; t < D / 16; ++t)
#pragma unroll
            for (int u = 0; u < 4; ++u) zacc[n][t][u] = 0.f;
    }
    uint32_t qb[NT][D / 16][2];

    for (int ch = 0; ch < nchunks; ++ch) {
        const int buf = ch & 1;
        if (ch + 1 < nchunks) load_block(buf ^ 1, ch + 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        if (ch == 0) {
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const char* qbase = reinterpret_cast<const char*>(sm.q[warp][n]);
                    qb[n][ks][0] = *reinterpret_cast<const uint32_t*>(qbase + swz<D>(g, 2 * ks) + c4 * 4);
                    qb[n][ks][1] = *reinterpret_cast<const uint32_t*>(qbase + swz<D>(g, 2 * ks + 1) + c4 * 4);
                }
        }
        float s[NT][CHUNK / 16][4];
        const uint32_t kb = smem_u32(sm.k[buf]);
#pragma unroll
        for (int mt = 0; mt < CHUNK / 16; ++mt) {
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int u = 0; u < 4; ++u) s[n][mt][u] = 0.f;
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
                const int mi = lane >> 3;
                const int row = mt * 16 + (mi & 1) * 8 + (lane & 7);
                const int chk = ks * 2 + (mi >> 1);
                uint32_t a0, a1, a2, a3;
                ldsm_x4(kb + swz<D>(row, chk), a0, a1, a2, a3);
#pragma unroll
                for (int n = 0; n < NT; ++n) mma16816(s[n][mt], a0, a1, a2, a3, qb[n][ks][0], qb[n][ks][1]);
            }
        }
        constexpr int PW = CHUNK + 8;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            float cmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
            for (int mt = 0; mt < CHUNK / 16; ++mt)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float x = s[n][mt][u] * sl2;
                    s[n][mt][u] = x;
                    cmax[u & 1] = fmaxf(cmax[u & 1], x);
                }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 4));
                cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 8));
                cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 16));
            }
            float corr[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float mn = fmaxf(m_run[n][h], cmax[h]);
                corr[h] = m_run[n][h] == -INFINITY ? 0.f : fast_ex2(m_run[n][h] - mn);
                m_run[n][h] = mn;
                l_part[n][h] *= corr[h];
            }
#pragma unroll
            for (int t = 0; t < D / 16; ++t) {
                zacc[n][t][0] *= corr[0];
                zacc[n][t][1] *= corr[1];
                zacc[n][t][2] *= corr[0];
                zacc[n][t][3] *= corr[1];
            }
#pragma unroll
            for (int mt = 0; mt < CHUNK / 16; ++mt)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float pv = fast_ex2(s[n][mt][u] - m_run[n][u & 1]);
                    l_part[n][u & 1] += pv;
                    sm.p[warp][n][(2 * c4 + (u & 1)) * PW + mt * 16 + g + (u >> 1) * 8] = __float2bfloat16_rn(pv);
                }
        }
        __syncwarp();
        const uint32_t vb = smem_u32(sm.v[buf]);
#pragma unroll
        for (int ks = 0; ks < CHUNK / 16; ++ks) {
            uint32_t b0[NT], b1[NT];
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                b0[n] = *reinterpret_cast<const uint32_t*>(&sm.p[warp][n][g * PW + ks * 16 + 2 * c4]);
                b1[n] = *reinterpret_cast<const uint32_t*>(&sm.p[warp][n][g * PW + ks * 16 + 8 + 2 * c4]);
            }
#pragma unroll
            for (int mt = 0; mt < D / 16; ++mt) {
                const int mi = lane >> 3;
                const int row = ks * 16 + (mi >> 1) * 8 + (lane & 7);
                const int chk = mt * 2 + (mi & 1);
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(vb + swz<D>(row, chk), a0, a1, a2, a3);
#pragma unroll
                for (int n = 0; n < NT; ++n) mma16816(zacc[n][mt], a0, a1, a2, a3, b0[n], b1[n]);
            }
        }
        __syncthreads();  // every warp done with `buf` before it is refilled
    }
    cp_async_wait<0>();
#pragma unroll
    for (int n = 0; n < NT; ++n) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            l_part[n][h] += __shfl_xor_sync(0xffffffffu, l_part[n][h], 4);
            l_part[n][h] += __shfl_xor_sync(0xffffffffu, l_part[n][h], 8);
            l_part[n][h] += __shfl_xor_sync(0xffffffffu, l_part[n][h], 16);
        }
        const float inv0 = l_part[n][0] > 0.f ? 1.f / l_part[n][0] : 0.f;
        const float inv1 = l_part[n][1] > 0.f ? 1.f / l_part[n][1] : 0.f;
        __nv_bfloat16* sq = sm.q[warp][n];
#pragma unroll
        for (int mt = 0; mt < D / 16; ++mt) {
            const int d0 = mt * 16 + g;
            sq[(2 * c4) * D + d0] = __float2bfloat16_rn(zacc[n][mt][0] * inv0);
            sq[(2 * c4 + 1) * D + d0] = __float2bfloat16_rn(zacc[n][mt][1] * inv1);
            sq[(2 * c4) * D + d0 + 8] = __float2bfloat16_rn(zacc[n][mt][2] * inv0);
            sq[(2 * c4 + 1) * D + d0 + 8] = __float2bfloat16_rn(zacc[n][mt][3] * inv1);
        }
    }
    __syncwarp();
    for (int t = lane; t < NT * 8 * kChunks16; t += 32) {
        const int n = t / (8 * kChunks16), rc = t % (8 * kChunks16);
        const int r = rc / kChunks16, c = rc % kChunks16;
        *reinterpret_cast<uint4*>(Z + (pair * L + r0 + n * 8 + r) * D + c * 8) =
            *reinterpret_cast<const uint4*>(&sm.q[warp][n][r * D + c * 8]);
    }
}

// The same block-row kernel with every kept block's K and V rows brought in
// by TMA (2-D tensor maps over [pairs L][d], 32-row x 64-column boxes,
// 128-byte swizzle; one thread issues 2 d/64 boxes per block and tensor)
// into a kStg-stage ring with full barriers, instead of 16-byte cp.async
// from every thread: the per-thread LDGSTS stream (256 per thread per block
// row at d = 128) and its L1 wavefronts are what bound the cp.async kernel
// (L1/TEX 71 %, L2 32 %, profiles/r02s_ncu_full_c3_block.txt).  ldmatrix
// reads the swizzled panels: chunk c of row r at (c / 8) 4 KB + r 128 +
// ((c % 8) ^ (r % 8)) 16.
template <int D, int NT, int kStg>
struct BlockSmemT {
    static constexpr int kWarps = 4 / NT;
    static constexpr int kHalf = 32 * 128;      // one 32-row x 64-column panel
    static constexpr int kKV = D / 64 * kHalf;  // K (or V) of one block
    unsigned char ring[kStg][2][kKV];           // [stage][K, V][panels]; Z staging at the end
    uint64_t full[kStg];
    static_assert(kStg * 2 * kKV >= kWarps * NT * 8 * D * 2, "Z staging fits the ring");
};

__device__ __forceinline__ uint32_t swz_panel(int r, int c) {
    return static_cast<uint32_t>((c >> 3) * (32 * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

template <int D, int NT, int kStg>
__global__ void __launch_bounds__(128 / NT)
    attn_block_tma_kernel(const __grid_constant__ CUtensorMap map_k, const __grid_constant__ CUtensorMap map_v,
                          const __nv_bfloat16* __restrict__ Q, const uint32_t* __restrict__ block_cols, int64_t L,
                          int64_t keep, int scale, __nv_bfloat16* __restrict__ Z) {
    constexpr int CHUNK = 32;
    extern __shared__ __align__(1024) unsigned char dsm[];
    using SM = BlockSmemT<D, NT, kStg>;
    SM& sm = *reinterpret_cast<SM*>(dsm);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nbr = L / 32;
    const int64_t pair = blockIdx.y, br = blockIdx.x;
    const int64_t r0 = br * 32 + warp * 8 * NT;  // this warp's first row
    const uint32_t* cols = block_cols + (pair * nbr + br) * keep;
    const int g = lane >> 2, c4 = lane & 3;
    constexpr int kChunks16 = D / 8;
    const int nchunks = static_cast<int>(keep);

    auto issue = [&](int ch) {  // one thread: block ch's K and V panels into stage ch % kStg
        const int st = ch % kStg;
        const int row = static_cast<int>(pair * L + static_cast<int64_t>(__ldg(cols + ch)) * 32);
        tc::mbar_expect_tx(&sm.full[st], 2 * SM::kKV);
#pragma unroll
        for (int h = 0; h < D / 64; ++h) {
            tc::tma_load_2d(tc::smem_addr(sm.ring[st][0] + h * SM::kHalf), &map_k, h * 64, row, &sm.full[st]);
            tc::tma_load_2d(tc::smem_addr(sm.ring[st][1] + h * SM::kHalf), &map_v, h * 64, row, &sm.full[st]);
        }
    };
    if (tid == 0) {
        for (int i = 0; i < kStg; ++i) tc::mbar_init(&sm.full[i], 1);
        tc::fence_barrier_init();
        for (int ch = 0; ch < kStg - 1 && ch < nchunks; ++ch) issue(ch);
    }
    // Q^T B fragments straight from global memory (row g of each band)
    uint32_t qb[NT][D / 16][2];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        const __nv_bfloat16* qr = Q + (pair * L + r0 + n * 8 + g) * D + c4 * 2;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
            qb[n][ks][0] = __ldg(reinterpret_cast<const unsigned int*>(qr + ks * 16));
            qb[n][ks][1] = __ldg(reinterpret_cast<const unsigned int*>(qr + ks * 16 + 8));
        }
    }

    const float sl2 = (scale ? rsqrtf(static_cast<float>(D)) : 1.f) * 1.4426950408889634f;
    float m_run[NT][2], l_part[NT][2];
    float zacc[NT][D / 16][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        m_run[n][0] = m_run[n][1] = -INFINITY;
        l_part[n][0] = l_part[n][1] = 0.f;
#pragma unroll
        for (int t = 0; t < D / 16; ++t)
#pragma unroll
            for (int u = 0; u < 4; ++u) zacc[n][t][u] = 0.f;
    }
    __syncthreads();  // the barriers are initialised

    for (int ch = 0; ch < nchunks; ++ch) {
        const int st = ch % kStg;
        // stage (ch + kStg - 1) % kStg held block ch - 1, released by the
        // barrier that ended the previous iteration
        if (tid == 0 && ch + kStg - 1 < nchunks) issue(ch + kStg - 1);
        tc::mbar_wait(&sm.full[st], (ch / kStg) & 1);
        float s[NT][CHUNK / 16][4];
        const uint32_t kb = tc::smem_addr(sm.ring[st][0]);
#pragma unroll
        for (int mt = 0; mt < CHUNK / 16; ++mt) {
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int u = 0; u < 4; ++u) s[n][mt][u] = 0.f;
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
                const int mi = lane >> 3;
                const int row = mt * 16 + (mi & 1) * 8 + (lane & 7);
                const int chk = ks * 2 + (mi >> 1);
                uint32_t a0, a1, a2, a3;
                ldsm_x4(kb + swz_panel(row, chk), a0, a1, a2, a3);
#pragma unroll
                for (int n = 0; n < NT; ++n) mma16816(s[n][mt], a0, a1, a2, a3, qb[n][ks][0], qb[n][ks][1]);
            }
        }
        // P^T as MMA B fragments straight from the S^T accumulators (movmatrix: no shared-memory round trip)
        uint32_t pb[NT][CHUNK / 16][2];
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            float cmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
            for (int mt = 0; mt < CHUNK / 16; ++mt)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float x = s[n][mt][u] * sl2;
                    s[n][mt][u] = x;
                    cmax[u & 1] = fmaxf(cmax[u & 1], x);
                }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 4));
                cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 8));
                cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 16));
            }
            float corr[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float mn = fmaxf(m_run[n][h], cmax[h]);
                corr[h] = m_run[n][h] == -INFINITY ? 0.f : fast_ex2(m_run[n][h] - mn);
                m_run[n][h] = mn;
                l_part[n][h] *= corr[h];
            }
#pragma unroll
            for (int t = 0; t < D / 16; ++t) {
                zacc[n][t][0] *= corr[0];
                zacc[n][t][1] *= corr[1];
                zacc[n][t][2] *= corr[0];
                zacc[n][t][3] *= corr[1];
            }
#pragma unroll
            for (int mt = 0; mt < CHUNK / 16; ++mt) {
                float pv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    pv[u] = fast_ex2(s[n][mt][u] - m_run[n][u & 1]);
                    l_part[n][u & 1] += pv[u];
                }
                pb[n][mt][0] = bc::movm_t(bc::pack_bf16(pv[0], pv[1]));  // keys g: -> P^T[keys 2c4, 2c4+1][query g]
                pb[n][mt][1] = bc::movm_t(bc::pack_bf16(pv[2], pv[3]));  // keys g + 8
            }
        }
        const uint32_t vb = tc::smem_addr(sm.ring[st][1]);
#pragma unroll
        for (int ks = 0; ks < CHUNK / 16; ++ks) {
            uint32_t b0[NT], b1[NT];
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                b0[n] = pb[n][ks][0];
                b1[n] = pb[n][ks][1];
            }
#pragma unroll
            for (int mt = 0; mt < D / 16; ++mt) {
                const int mi = lane >> 3;
                const int row = ks * 16 + (mi >> 1) * 8 + (lane & 7);
                const int chk = mt * 2 + (mi & 1);
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(vb + swz_panel(row, chk), a0, a1, a2, a3);
#pragma unroll
                for (int n = 0; n < NT; ++n) mma16816(zacc[n][mt], a0, a1, a2, a3, b0[n], b1[n]);
            }
        }
        __syncthreads();  // every warp done with stage `st` before it is refilled
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            l_part[n][h] += __shfl_xor_sync(0xffffffffu, l_part[n][h], 4);
            l_part[n][h] += __shfl_xor_sync(0xffffffffu, l_part[n][h], 8);
            l_part[n][h] += __shfl_xor_sync(0xffffffffu, l_part[n][h], 16);
        }
        const float inv0 = l_part[n][0] > 0.f ? 1.f / l_part[n][0] : 0.f;
        const float inv1 = l_part[n][1] > 0.f ? 1.f / l_part[n][1] : 0.f;
        // Z staged in the (now idle) ring: this warp's [NT][8][D] slab
        __nv_bfloat16* sq = reinterpret_cast<__nv_bfloat16*>(&sm.ring[0][0][0]) + (warp * NT + n) * 8 * D;
#pragma unroll
        for (int mt = 0; mt < D / 16; ++mt) {
            const int d0 = mt * 16 + g;
            sq[(2 * c4) * D + d0] = __float2bfloat16_rn(zacc[n][mt][0] * inv0);
            sq[(2 * c4 + 1) * D + d0] = __float2bfloat16_rn(zacc[n][mt][1] * inv1);
            sq[(2 * c4) * D + d0 + 8] = __float2bfloat16_rn(zacc[n][mt][2] * inv0);
            sq[(2 * c4 + 1) * D + d0 + 8] = __float2bfloat16_rn(zacc[n][mt][3] * inv1);
        }
    }
    __syncwarp();
    const __nv_bfloat16* zs = reinterpret_cast<const __nv_bfloat16*>(&sm.ring[0][0][0]) + warp * NT * 8 * D;
    for (int t = lane; t < NT * 8 * kChunks16; t += 32) {
        const int n = t / (8 * kChunks16), rc = t % (8 * kChunks16);
        const int r = rc / kChunks16, c = rc % kChunks16;
        *reinterpret_cast<uint4*>(Z + (pair * L + r0 + n * 8 + r) * D + c * 8) =
            *reinterpret_cast<const uint4*>(&zs[(n * 8 + r) * D + c * 8]);
    }
}

template <int D, int NT, int kStg>
void launch_block_tma(const AttnArgs& a, cudaStream_t st) {
    const size_t smem = sizeof(BlockSmemT<D, NT, kStg>) + 1024;
    auto kern = attn_block_tma_kernel<D, NT, kStg>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const CUtensorMap mk = make_map(a.k, a.pairs * a.L, D, 32, 64);
    const CUtensorMap mv = make_map(a.v, a.pairs * a.L, D, 32, 64);
    const dim3 grid(static_cast<unsigned>(a.L / 32), static_cast<unsigned>(a.pairs));
    kern<<<grid, 128 / NT, smem, st>>>(mk, mv, static_cast<const __nv_bfloat16*>(a.q), a.cols, a.L, a.keep, a.scale,
                                       static_cast<__nv_bfloat16*>(a.z));
}

template <int D, int NT>
void launch_block_nt(const AttnArgs& a, cudaStream_t st) {
    const size_t smem = sizeof(BlockSmemN<D, NT>);
    auto kern = attn_block_nt_kernel<D, NT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const dim3 grid(static_cast<unsigned>(a.L / 32), static_cast<unsigned>(a.pairs));
    kern<<<grid, 128 / NT, smem, st>>>(static_cast<const __nv_bfloat16*>(a.q), static_cast<const __nv_bfloat16*>(a.k),
                                       static_cast<const __nv_bfloat16*>(a.v), a.cols, a.L, a.keep, a.scale,
                                       static_cast<__nv_bfloat16*>(a.z));
}

// ---------------------------------------------------------------- v2
// K fragments straight from global memory into registers: the reduction
// order over d is permuted so each lane's slots of a k-step are 4 CONSECUTIVE
// d values of one 32/64-byte row segment (16-byte loads, no shared memory,
// no ldmatrix); the Q^T B-fragments use the same permutation.  One index
// load per gathered row (lane = row, shared by shuffles).  V rows still go
// through cp.async + XOR-swizzled shared memory for ldmatrix.trans.
// MODE kBandList: COLVEC -- the warp's 8 query rows share one key list.
// MODE kRowsBand: every query row has its own list (ROW_TOPK rows of `keep`,
//   THRESHOLD CSR rows); a warp takes 8 consecutive rows
//   and streams the CONCATENATION of their lists (contiguous in the CSR /
//   row-list layout) in 32-key chunks, each row in its own MMA column; an
//   entry (key, column) is live only when the key's stream position lies in
//   that row's segment.  No per-row latency chain: one long prefetched
//   gather stream per warp (the MMA does 8x the useful work, which is free).
enum BandMode { kBandList = 0, kRowsBand = 4 };

template <int D, int kWarps, int MODE>
__global__ void __launch_bounds__(kWarps * 32)
    attn_band_v2_kernel(const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ K,
                        const __nv_bfloat16* __restrict__ V, const uint32_t* __restrict__ band_cols,
                        int64_t pairs, int64_t L, int64_t keep, int scale, __nv_bfloat16* __restrict__ Z,
                        const uint64_t* __restrict__ rowptr, uint8_t* __restrict__ empty_rows) {
    constexpr int CH = 32;
    constexpr int NW = D / 32;        // uint4 per lane per K row segment (D/4 bf16)
    constexpr int kRows = 8;  // query rows per warp
    extern __shared__ __align__(128) unsigned char dsm[];
    using S = BandSmemV2<D>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    S& sm = reinterpret_cast<S*>(dsm)[warp];
    constexpr bool SEG = MODE == kRowsBand;
    const int64_t nb = (L + 7) / 8;  // warp work items (bands) per pair
    const int64_t band_global = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
    if (band_global >= pairs * nb) return;
    const int64_t pair = band_global / nb, band = band_global % nb;
    const int64_t r0 = band * kRows;
    const __nv_bfloat16* Kp = K + pair * L * D;
    const __nv_bfloat16* Vp = V + pair * L * D;
    const uint32_t* cols = band_cols + (pair * nb + band) * keep;
    int64_t nkeys = keep;
    const int g = lane >> 2, c4 = lane & 3;
    // kRowsBand: stream segment bounds of this thread's two columns (rows
    // 2c4, 2c4+1): [sb0, sb1) and [sb1, sb2)
    int64_t sb0 = 0, sb1 = 0, sb2 = 0;
    if (SEG) {
        const int64_t e = r0 + 8 < L ? r0 + 8 : L;
        auto bound = [&](int c) -> int64_t {
            const int64_t r = r0 + c < e ? r0 + c : e;
            return rowptr ? static_cast<int64_t>(rowptr[pair * L + r]) : (pair * L + r) * keep;
        };
        const int64_t b0 = bound(0);
        cols = band_cols + b0;
        nkeys = bound(8) - b0;
        sb0 = bound(2 * c4) - b0;
        sb1 = bound(2 * c4 + 1) - b0;
        sb2 = bound(2 * c4 + 2) - b0;
    }
    auto chunk_idx = [&](int ch) -> uint32_t {
        const int64_t p = static_cast<int64_t>(ch) * CH + lane;
        return p < nkeys ? __ldg(cols + p) : 0u;
    };
    band_core<D, kRows, SEG>(sm, Q, Kp, Vp, pair, L, r0, nkeys, sb0, sb1, sb2, scale, Z, chunk_idx, lane);
    if (SEG && empty_rows && g == 0) {
        if (r0 + 2 * c4 < L) empty_rows[pair * L + r0 + 2 * c4] = sb1 == sb0;
        if (r0 + 2 * c4 + 1 < L) empty_rows[pair * L + r0 + 2 * c4 + 1] = sb2 == sb1;
    }
}

template <int D, int kWarps, int MODE = kBandList>
void launch_band_v2(const AttnArgs& a, cudaStream_t st) {
    const int64_t nb = (a.L + 7) / 8;
    const size_t smem = sizeof(BandSmemV2<D>) * kWarps;
    auto kern = attn_band_v2_kernel<D, kWarps, MODE>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const unsigned grid = static_cast<unsigned>(ceil_div_i(a.pairs * nb, kWarps));
    kern<<<grid, kWarps * 32, smem, st>>>(
        static_cast<const __nv_bfloat16*>(a.q), static_cast<const __nv_bfloat16*>(a.k),
        static_cast<const __nv_bfloat16*>(a.v), a.cols, a.pairs, a.L, a.keep, a.scale,
        static_cast<__nv_bfloat16*>(a.z), a.rowptr, a.empty_rows);
}

}  // namespace

bool band_attention_supported(const AttnArgs& a) {
    if (!a.bf16 || (a.D != 64 && a.D != 128)) return false;
    if (options().attn_generic) return false;  // parity tests of the generic kernel
    if (a.mode == kColvec) return a.vec_v == 8;
    if (a.mode == kRowTopk || a.mode == kThreshold) return true;
    return a.mode == kBlock && a.block == 32 && a.L % 32 == 0;  // block rows = 4 bands
}

void run_band_attention(const AttnArgs& a, cudaStream_t st) {
    if (a.mode == kBlock) {
        if (options().block_cpasync) {
            if (a.D == 64) launch_block_nt<64, 2>(a, st);
            else launch_block_nt<128, 2>(a, st);
        } else {
            if (a.D == 64) launch_block_tma<64, 2, BLK_STAGES>(a, st);
            else launch_block_tma<128, 2, BLK_STAGES>(a, st);
        }
    } else if (a.mode == kRowTopk || a.mode == kThreshold) {
        AttnArgs b = a;
        if (a.mode == kRowTopk) b.rowptr = nullptr;  // fixed-length row lists
        if (a.D == 64) launch_band_v2<64, 16, kRowsBand>(b, st);
        else launch_band_v2<128, 8, kRowsBand>(b, st);
    } else {
        if (a.D == 64) launch_band_v2<64, 16>(a, st);
        else launch_band_v2<128, 8>(a, st);
    }
    note_launch();
}

}  // namespace dsa
