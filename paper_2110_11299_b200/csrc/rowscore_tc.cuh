// Row-owner tensor-core score streaming shared by the per-row selection
// kernels (threshold, per-row top-k): one CTA of 128 threads owns 128 query
// rows (thread = row = TMEM lane); score_pass() streams the K~ tiles of 64
// keys through tcgen05.mma (M = 128 queries, N = 64 keys, K = k) into a
// double-buffered TMEM accumulator and hands each thread its row's 32-score
// column groups.  Levels are chunk-planar ([k/8][L][8] per pair).
#pragma once

#include <stdint.h>

#include "device_common.cuh"
#include "tc_sm100.cuh"

namespace dsa {
namespace rs {

constexpr int kTQ = 128;  // query rows per CTA (UMMA M) = threads
constexpr int kTN = 64;   // keys per tile (UMMA N)
constexpr int kSt = 3;    // K~ tile ring
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// K-major no-swizzle canonical layout (8-row x 16-byte cores, LBO = 128,
// SBO = KD * 16), filled from the chunk-planar levels: consecutive threads
// copy consecutive rows of one 8-column chunk (contiguous in HBM).
template <int KD>
__device__ __forceinline__ uint32_t toff(int r, int c) {
    return static_cast<uint32_t>((r >> 3) * (KD * 16) + c * 128 + (r & 7) * 16);
}
template <int KD, int ROWS>
__device__ __forceinline__ void load_rows(uint32_t sbase, const uint16_t* __restrict__ src, int64_t row0,
                                          int64_t L, int tid) {
    constexpr int kCh = KD / 8;
    for (int t = tid; t < ROWS * kCh; t += kTQ) {
        const int c = t / ROWS, r = t % ROWS;
        const bool ok = row0 + r < L;
        cp16(sbase + toff<KD>(r, c), src + lvl_index(L, ok ? (row0 + r) : 0, c * 8), ok);
    }
}

struct PassCtx {
    unsigned char* ring;
    uint64_t* bars;
    uint32_t tmem;
    uint64_t qdesc;
    const uint16_t* lkp;
    int64_t L;
    int nkt;
    int tid, warp;
};

// Streams key tiles 0..nkt-1 through the tensor core and calls
// f(tile, regs, col0) with 32 score columns of this thread's row.  `g`
// counts tiles over all passes (TMEM buffer + mbarrier phase).
template <int KD, class F>
__device__ __forceinline__ void score_pass(const PassCtx& c, uint32_t& g, F&& f) {
    constexpr int kTile = kTN * KD * 2;
    constexpr uint32_t idesc = tc::idesc_bf16_f32(kTQ, kTN);
    for (int s = 0; s < kSt; ++s) {
        if (s < c.nkt) load_rows<KD, kTN>(tc::smem_addr(c.ring + s * kTile), c.lkp, static_cast<int64_t>(s) * kTN, c.L, c.tid);
        cp_commit();
    }
    for (int t = 0; t <= c.nkt; ++t) {
        if (t >= 1) {
            const uint32_t u = g + t - 1;
            tc::mbar_wait(&c.bars[u & 1], (u >> 1) & 1);
            tc::fence_after_sync();
            const int nxt = t - 1 + kSt;
            if (nxt < c.nkt)
                load_rows<KD, kTN>(tc::smem_addr(c.ring + ((t - 1) % kSt) * kTile), c.lkp,
                                   static_cast<int64_t>(nxt) * kTN, c.L, c.tid);
            cp_commit();
        }
        if (t < c.nkt) {
            cp_wait<kSt - 1>();
            tc::fence_proxy_async();
            __syncthreads();
            if (c.tid == 0) {
                tc::fence_after_sync();
                const uint32_t bbase = tc::smem_addr(c.ring + (t % kSt) * kTile);
#pragma unroll
                for (int ks = 0; ks < KD / 16; ++ks) {
                    const uint64_t bd = tc::desc_kmajor_nosw(bbase + ks * 256, 128, KD * 16);
                    const uint64_t ad = c.qdesc + static_cast<uint64_t>((ks * 256) >> 4);
                    tc::mma_bf16(c.tmem + ((g + t) & 1) * kTN, ad, bd, idesc, ks > 0);
                }
                tc::commit(&c.bars[(g + t) & 1]);
            }
        }
        if (t >= 1) {
            const int u = t - 1;
            const uint32_t base = c.tmem + (static_cast<uint32_t>(c.warp * 32) << 16) + ((g + u) & 1) * kTN;
            uint32_t r0[32], r1[32];
            tc::ld_32x32b_x32(base, r0);
            tc::ld_32x32b_x32(base + 32, r1);
            tc::wait_ld();
            f(u, r0, 0);
            f(u, r1, 32);
            tc::fence_before_sync();
        }
        __syncthreads();
    }
    cp_wait<0>();
    g += static_cast<uint32_t>(c.nkt);
}

}  // namespace rs
}  // namespace dsa
