// Phase 2 for vector-wise masks (COLVEC, v = 8), warp-specialised and
// persistent: the TMEM-bound score / max-pool epilogue of one 64-query block
// overlaps the ALU-bound exact selection of the previous block.
//
// Roles (26 warps, one CTA per SM, work items = (pair, 64-query block)):
//   warp 0      producer (one lane): bulk copies (TMA engine) of K~ tiles
//               (128 keys) into an 8-slot ring and the item's Q~ block;
//               completion (tx bytes) -> tile_full[slot]
//   warp 1      MMA issuer (one lane): tcgen05.mma kind::f16, M = 128 keys,
//               N = 64 queries, K = 16 (one instruction per tile) into a
//               double-buffered TMEM accumulator; tcgen05.commit ->
//               tmem_full[buf] and slot_free[slot]
//   warps 2-9   epilogue: tcgen05.ld 32x32b (thread = key), band max over 8
//               columns in registers (FMNMX3), pooled int16 scores into a
//               double-buffered shared array; -> tmem_empty, pooled_full
//   warps 10-25 selection: two warps per band (column halves, private
//               histograms merged through a pair barrier), exact threshold
//               + ascending emission; -> pooled_empty
// The fp32 accumulator holds the exact integer score (levels <= 7 in bf16,
// |S| < 2^24); ties resolve to the lowest column (P/src/linalg.cpp:77-80).
#include <cuda_bf16.h>

#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"
#include "select_common.cuh"
#include "tc_sm100.cuh"

namespace dsa {
namespace {

using namespace sel;

constexpr int kNQ = 64;        // queries per work item (8 bands)
constexpr int kMT = 128;       // keys per tile
constexpr int kStages = 8;
constexpr int kAcc = 4;       // TMEM accumulator buffers (kAcc * kNQ columns)
constexpr int kWarps = 26;
constexpr int kThreads = kWarps * 32;
constexpr int kEpi0 = 2, kSel0 = 10;  // 8 epilogue warps (lane quarter, column half), 16 selection warps

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int KD>
__device__ __forceinline__ uint32_t tile_off(int r, int chunk16) {
    return static_cast<uint32_t>((r >> 3) * (KD * 16) + chunk16 * 128 + (r & 7) * 16);
}

// TMA-engine bulk copy global -> shared, completion counted on `bar` (tx bytes)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            tc::smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(tc::smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tc::smem_addr(bar)), "r"(bytes)
                 : "memory");
}

struct WsBars {
    uint64_t tile_full[kStages], slot_free[kStages];
    uint64_t tmem_full[kAcc], tmem_empty[kAcc];
    uint64_t pooled_full[2], pooled_empty[2];
    uint32_t tmem_slot;
};

template <int KD>
__global__ void __launch_bounds__(kThreads, 1)
    colvec_ws_kernel(const uint16_t* __restrict__ lq, const uint16_t* __restrict__ lk, int64_t pairs,
                     int64_t L, int64_t keep, int M, uint32_t* __restrict__ out, int dbg) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int kTileA = kMT * KD * 2, kTileB = kNQ * KD * 2;
    const int nt = static_cast<int>((L + kMT - 1) / kMT);
    const int Lp = nt * kMT;
    const int64_t nblk = (L + kNQ - 1) / kNQ;
    const int64_t items = pairs * nblk;
    const int64_t nb = (L + 7) / 8;

    unsigned char* p = smem;
    unsigned char* ring = p;   p += kStages * kTileA;
    unsigned char* qbuf = p;   p += 2 * kTileB;
    int16_t* pooled = reinterpret_cast<int16_t*>(p); p += 2 * 8 * Lp * 2;
    uint32_t* hist = reinterpret_cast<uint32_t*>(p); p += (16 * 64 + 8 * kWin) * 4;  // pair hists + fallback
    uint32_t* obufs = reinterpret_cast<uint32_t*>(p); p += 8 * kList * 4;
    int* bandmax = reinterpret_cast<int*>(p); p += 2 * 8 * 4;
    WsBars& bar = *reinterpret_cast<WsBars*>(p);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&bar.tile_full[s], 1);
            tc::mbar_init(&bar.slot_free[s], 1);
        }
        for (int b = 0; b < kAcc; ++b) {
            tc::mbar_init(&bar.tmem_full[b], 1);
            tc::mbar_init(&bar.tmem_empty[b], 8);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&bar.pooled_full[b], 8);
            tc::mbar_init(&bar.pooled_empty[b], 16);
        }
        tc::fence_barrier_init();
    }
    if (tid < 16) bandmax[tid] = INT32_MIN;
    if (warp == 1) tc::tmem_alloc<kAcc * kNQ>(&bar.tmem_slot);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = bar.tmem_slot;
    // this CTA's work items: blockIdx.x, +gridDim.x, ...
    const int64_t my_items = items > blockIdx.x ? (items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t total_tiles = my_items * nt;

    if (warp == 0) {
        // ---------------------------------------------------------- producer
        // Levels are chunk-planar ([KD/8][L][8] per pair), so each 8-column
        // plane of a tile is one contiguous run: KD/8 bulk copies per tile
        // (+ KD/8 for the item's Q~ block), all issued by one lane.
        if (lane == 0) {
            for (int64_t g = 0; g < total_tiles; ++g) {
                const int64_t n = g / nt;
                const int t = static_cast<int>(g % nt);
                const int64_t item = blockIdx.x + n * gridDim.x;
                const int64_t pair = item / nblk;
                const int slot = static_cast<int>(g % kStages);
                if (g >= kStages) tc::mbar_wait(&bar.slot_free[slot], static_cast<uint32_t>((g / kStages - 1) & 1));
                const int64_t row0 = static_cast<int64_t>(t) * kMT;
                const uint32_t rows = static_cast<uint32_t>(L - row0 < kMT ? L - row0 : kMT);
                const int64_t q0 = (item % nblk) * kNQ;
                const uint32_t qrows = static_cast<uint32_t>(L - q0 < kNQ ? L - q0 : kNQ);
                const uint32_t bytes = (KD / 8) * rows * 16 + (t == 0 ? (KD / 8) * qrows * 16 : 0);
                arrive_expect_tx(&bar.tile_full[slot], bytes);
                if (t == 0) {
#pragma unroll
                    for (int c = 0; c < KD / 8; ++c)
                        bulk_g2s(qbuf + (n & 1) * kTileB + c * (kNQ * 16), lq + pair * L * KD + (c * L + q0) * 8,
                                 qrows * 16, &bar.tile_full[slot]);
                }
#pragma unroll
                for (int c = 0; c < KD / 8; ++c)
                    bulk_g2s(ring + slot * kTileA + c * (kMT * 16), lk + pair * L * KD + (c * L + row0) * 8,
                             rows * 16, &bar.tile_full[slot]);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // --------------------------------------------------------------- MMA
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_bf16_f32(kMT, kNQ);
            for (int64_t g = 0; g < total_tiles; ++g) {
                const int64_t n = g / nt;
                const int slot = static_cast<int>(g % kStages);
                const int buf = static_cast<int>(g % kAcc);
                tc::mbar_wait(&bar.tile_full[slot], static_cast<uint32_t>((g / kStages) & 1));
                if (g >= kAcc) tc::mbar_wait(&bar.tmem_empty[buf], static_cast<uint32_t>((g / kAcc - 1) & 1));
                tc::fence_after_sync();
                const uint32_t abase = tc::smem_addr(ring + slot * kTileA);
                const uint32_t bbase = tc::smem_addr(qbuf + (n & 1) * kTileB);
                if (dbg & 4) {  // profiling switch: no MMA
                    tc::mbar_arrive(&bar.tmem_full[buf]);
                    tc::mbar_arrive(&bar.slot_free[slot]);
                    continue;
                }
#pragma unroll
                for (int ks = 0; ks < KD / 16; ++ks)
                    tc::mma_bf16(tmem + buf * kNQ, tc::desc_kmajor_nosw(abase + ks * 2 * (kMT * 16), kMT * 16, 128),
                                 tc::desc_kmajor_nosw(bbase + ks * 2 * (kNQ * 16), kNQ * 16, 128), idesc, ks > 0);
                tc::commit(&bar.tmem_full[buf]);
                tc::commit(&bar.slot_free[slot]);
            }
        }
        __syncwarp();
    } else if (warp < kSel0) {
        // ---------------------------------------------------------- epilogue
        const int quarter = warp & 3, half = (warp - kEpi0) >> 2;  // columns [32*half, +32) = bands 4*half..+3
        for (int64_t n = 0; n < my_items; ++n) {
            const int64_t item = blockIdx.x + n * gridDim.x;
            const int64_t q0 = (item % nblk) * kNQ;
            const int pb = static_cast<int>(n & 1);
            if (n >= 2) tc::mbar_wait_sleep(&bar.pooled_empty[pb], static_cast<uint32_t>(((n >> 1) - 1) & 1));
            int16_t* pool = pooled + pb * 8 * Lp;
            const bool ragged_q = q0 + kNQ > L;
            float bmax[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) bmax[i] = -INFINITY;
            for (int t = 0; t < nt; ++t) {
                const int64_t g = n * nt + t;
                const int buf = static_cast<int>(g % kAcc);
                tc::mbar_wait(&bar.tmem_full[buf], static_cast<uint32_t>((g / kAcc) & 1));
                tc::fence_after_sync();
                const int key = t * kMT + quarter * 32 + lane;
                const bool kvalid = key < L;
                const uint32_t base = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + buf * kNQ + half * 32;
                uint32_t r0[32];
                if (dbg & 2) {  // profiling switch: no TMEM reads
#pragma unroll
                    for (int x = 0; x < 32; ++x) r0[x] = 0;
                } else {
                    tc::ld_32x32b_x32(base, r0);
                    tc::wait_ld();
                }
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bar.tmem_empty[buf]);
                {
                    uint32_t* r = r0;
                    if (ragged_q) {
#pragma unroll
                        for (int x = 0; x < 32; ++x)
                            if (q0 + half * 32 + x >= L) r[x] = __float_as_uint(-INFINITY);
                    }
#pragma unroll
                    for (int bb = 0; bb < 4; ++bb) {
                        float m0, m1, m2;
                        const float* f = reinterpret_cast<const float*>(&r[bb * 8]);
                        asm("max.f32 %0, %1, %2, %3;" : "=f"(m0) : "f"(f[0]), "f"(f[1]), "f"(f[2]));
                        asm("max.f32 %0, %1, %2, %3;" : "=f"(m1) : "f"(f[3]), "f"(f[4]), "f"(f[5]));
                        asm("max.f32 %0, %1, %2, %3;" : "=f"(m2) : "f"(m0), "f"(m1), "f"(f[6]));
                        const float mx = fmaxf(m2, f[7]);
                        const int band = half * 4 + bb;
                        pool[band * Lp + key] = kvalid ? static_cast<int16_t>(__float2int_rn(mx)) : INT16_MIN;
                        if (kvalid) bmax[bb] = fmaxf(bmax[bb], mx);
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float v = bmax[i];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
                if (lane == 0) atomicMax(&bandmax[pb * 8 + half * 4 + i], __float2int_rn(v));
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&bar.pooled_full[pb]);
        }
    } else {
        // --------------------------------------------------------- selection
        // two warps per band: part 0 owns columns [0, mid), part 1 [mid, Lp)
        const int sw = warp - kSel0, band_l = sw >> 1, part = sw & 1;
        const int mid = (nt / 2) * kMT;
        const int lo_col = part ? mid : 0, hi_col = part ? Lp : mid;
        uint32_t* h_own = hist + sw * 64;
        uint32_t* h_0 = hist + (band_l * 2) * 64;
        uint32_t* h_1 = hist + (band_l * 2 + 1) * 64;
        uint32_t* obuf = obufs + band_l * kList;
        const uint32_t kk = static_cast<uint32_t>(keep);
        const unsigned lt = lanemask_lt();
        for (int64_t n = 0; n < my_items; ++n) {
            const int64_t item = blockIdx.x + n * gridDim.x;
            const int64_t pair = item / nblk;
            const int64_t q0 = (item % nblk) * kNQ;
            const int pb = static_cast<int>(n & 1);
            tc::mbar_wait_sleep(&bar.pooled_full[pb], static_cast<uint32_t>((n >> 1) & 1));
            const int64_t band = q0 / 8 + band_l;
            const int16_t* pv = pooled + (pb * 8 + band_l) * Lp;
            const int bmax = bandmax[pb * 8 + band_l];
            const int lo = bmax - 63;
            // 1. private 64-bin histogram of this part's columns scoring >= lo
            h_own[lane] = 0;
            h_own[lane + 32] = 0;
            __syncwarp();
            for (int j0 = lo_col; j0 < hi_col; j0 += 128) {
                int v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = pv[j0 + u * 32 + lane];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (v[u] >= lo) atomicAdd(&h_own[v[u] - lo], 1u);
            }
            asm volatile("bar.sync %0, 64;\n" ::"r"(1 + band_l) : "memory");
            // 2. combined threshold (both warps compute the same T, rem)
            const uint32_t a0 = h_0[2 * lane], a1 = h_0[2 * lane + 1];
            const uint32_t c0 = a0 + h_1[2 * lane], c1 = a1 + h_1[2 * lane + 1];
            uint32_t tot = c0 + c1;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
            const bool fast = band < nb && tot >= kk && !(dbg & 1);
            if (fast) {
                const uint32_t local = c0 + c1;
                uint32_t suf = local;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t y = __shfl_down_sync(0xffffffffu, suf, off);
                    if (lane + off < 32) suf += y;
                }
                const uint32_t excl = suf - local;
                const bool mine = excl < kk && kk <= suf;
                const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
                int tb = 0;
                uint32_t r = 0;
                if (mine) {
                    if (excl + c1 >= kk) {
                        tb = 2 * lane + 1;
                        r = kk - excl;
                    } else {
                        tb = 2 * lane;
                        r = kk - excl - c1;
                    }
                }
                tb = __shfl_sync(0xffffffffu, tb, src);
                const uint32_t rem = __shfl_sync(0xffffffffu, r, src);
                const int T = lo + tb;
                // part 0 counts: values > T and == T among columns [0, mid)
                uint32_t gt0 = (2 * lane > tb ? a0 : 0u) + (2 * lane + 1 > tb ? a1 : 0u);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) gt0 += __shfl_xor_sync(0xffffffffu, gt0, off);
                const uint32_t eq0 = h_0[tb];
                const uint32_t eq0_take = eq0 < rem ? eq0 : rem;
                uint32_t taken = part ? gt0 + eq0_take : 0u;
                const uint32_t rem_p = part ? rem - eq0_take : eq0_take;
                uint32_t eq_seen = 0;
                // 3. ascending emission of this part into the band's staging list
                for (int j0 = lo_col; j0 < hi_col; j0 += 128) {
                    int v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[u] = pv[j0 + u * 32 + lane];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const bool eq = v[u] == T;
                        const unsigned be = vote_ballot(eq);
                        const bool take = v[u] > T || (eq && eq_seen + __popc(be & lt) < rem_p);
                        const unsigned bt = vote_ballot(take);
                        obuf[take ? taken + __popc(bt & lt) : static_cast<uint32_t>(kList - 32 + lane)] =
                            static_cast<uint32_t>(j0 + u * 32 + lane);
                        taken += __popc(bt);
                        eq_seen += __popc(be);
                    }
                }
            } else if (band < nb && part == 0 && !(dbg & 1)) {
                // rare: k-th value more than 63 below the band max -> full-band path
                band_select(pv, static_cast<int>(L), Lp, static_cast<int>(keep), bmax, M, hist + 16 * 64 + band_l * kWin, obuf,
                            out + (pair * nb + band) * keep, lane);
            }
            asm volatile("bar.sync %0, 64;\n" ::"r"(1 + band_l) : "memory");
            if (fast) {
                uint32_t* o = out + (pair * nb + band) * keep;
                for (int i = part * 32 + lane; i < keep; i += 64) o[i] = obuf[i];
            }
            asm volatile("bar.sync %0, 64;\n" ::"r"(1 + band_l) : "memory");
            if (lane == 0) {
                if (part == 0) bandmax[pb * 8 + band_l] = INT32_MIN;
                tc::mbar_arrive(&bar.pooled_empty[pb]);
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc<kAcc * kNQ>(tmem);
}

template <int KD>
size_t ws_smem_bytes(int64_t L) {
    const int64_t Lp = (L + kMT - 1) / kMT * kMT;
    return static_cast<size_t>(kStages * kMT * KD * 2 + 2 * kNQ * KD * 2 + 2 * 8 * Lp * 2 + (16 * 64 + 8 * kWin) * 4 +
                               8 * kList * 4 + 2 * 8 * 4) +
           sizeof(WsBars) + 16;
}

}  // namespace

bool colvec_ws_supported(const SelectArgs& a) {
    if (a.mode != kColvec || a.vec_v != 8 || a.per_row || a.qmax > 7) return false;
    if (a.KD != 16 && a.KD != 32) return false;
    if (a.keep > kList - 32) return false;
    if ((a.L + kMT - 1) / kMT < kStages) return false;  // Q~ double buffer needs >= kStages tiles per block
    const size_t smem = a.KD == 16 ? ws_smem_bytes<16>(a.L) : ws_smem_bytes<32>(a.L);
    return smem <= 227 * 1024;
}

void run_colvec_ws(const SelectArgs& a, cudaStream_t st) {
    // DSA_PROFILE_SWITCH (profiling-only ablations): 1 skip selection, 2 skip TMEM reads, 4 skip MMA
    static const int dbg = [] {
        const char* e = std::getenv("DSA_PROFILE_SWITCH");
        return e ? std::atoi(e) : 0;
    }();
    const int M = static_cast<int>(a.KD) * a.qmax * a.qmax;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t items = a.pairs * ceil_div_i(a.L, kNQ);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(items, sms));
    if (a.KD == 16) {
        const size_t smem = ws_smem_bytes<16>(a.L);
        cudaFuncSetAttribute(colvec_ws_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        colvec_ws_kernel<16><<<grid, kThreads, smem, st>>>(a.lq, a.lk, a.pairs, a.L, a.keep, M, a.cols, dbg);
    } else {
        const size_t smem = ws_smem_bytes<32>(a.L);
        cudaFuncSetAttribute(colvec_ws_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        colvec_ws_kernel<32><<<grid, kThreads, smem, st>>>(a.lq, a.lk, a.pairs, a.L, a.keep, M, a.cols, dbg);
    }
    note_launch();
}

}  // namespace dsa
