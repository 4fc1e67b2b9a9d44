// Row-owner tensor-core score streaming shared by the per-row selection
// kernels (threshold, per-row top-k): one CTA of 128 threads owns 128 query
// rows (thread = row = TMEM lane); score_pass() streams the K~ tiles of 64
// keys through tcgen05.mma (M = 128 queries, N = 64 keys, K = k) into a
// double-buffered TMEM accumulator and hands each thread its row's 32-score
// column groups.  Levels are chunk-planar ([k/8][L][8] per pair).
#pragma once

#include <cuda_fp16.h>
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
// PERM: key r of each 32-key group goes to tile row 2(r%16) + r/16, so a
// .pack::16b TMEM load of an f16 accumulator gives register i = (key i,
// key 16+i) of the group (bit i / bit 16+i of a packed compare mask = key
// order)
template <int KD, int ROWS, bool PERM = false>
__device__ __forceinline__ void load_rows(uint32_t sbase, const uint16_t* __restrict__ src, int64_t row0,
                                          int64_t L, int tid) {
    constexpr int kCh = KD / 8;
    for (int t = tid; t < ROWS * kCh; t += kTQ) {
        const int c = t / ROWS, r = t % ROWS;
        const bool ok = row0 + r < L;
        const int rd = PERM ? ((r & ~31) | ((r & 15) << 1) | ((r >> 4) & 1)) : r;
        cp16(sbase + toff<KD>(rd, c), src + lvl_index(L, ok ? (row0 + r) : 0, c * 8), ok);
    }
}

// In-place bf16 -> f16 conversion of the 16-byte pieces THIS thread copied
// with load_rows<KD, ROWS, PERM> (after its cp.async group completed): the
// levels are small integers, exact in both formats.  The f16-accumulator
// MMA (P16) needs f16 operands.
template <int KD, int ROWS, bool PERM = false>
__device__ __forceinline__ void cvt_rows_f16(unsigned char* sbase, int tid) {
    constexpr int kCh = KD / 8;
    for (int t = tid; t < ROWS * kCh; t += kTQ) {
        const int c = t / ROWS, r = t % ROWS;
        const int rd = PERM ? ((r & ~31) | ((r & 15) << 1) | ((r >> 4) & 1)) : r;
        uint4* q = reinterpret_cast<uint4*>(sbase + toff<KD>(rd, c));
        uint4 v = *q;
        uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xffff0000u);
            __half2 h = __floats2half2_rn(lo, hi);
            w[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        *q = v;
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
//
// P16 (exact only when every score and partial sum is an integer of
// magnitude <= 2048, i.e. KD * qmax^2 <= 2048): f16 operands (converted in
// shared memory, cvt_rows_f16; the caller converts the Q~ tile) and f16
// accumulator (bf16 operands need an f32 accumulator), key rows
// permuted (load_rows PERM) and ONE .pack::16b load per tile, so
// f(tile, regs, 0) gets 32 registers of f16 pairs: register i (i < 16) =
// (key i, key 16+i), register 16+i = (key 32+i, key 48+i).
template <int KD, bool P16 = false, class F>
__device__ __forceinline__ void score_pass(const PassCtx& c, uint32_t& g, F&& f) {
    constexpr int kTile = kTN * KD * 2;
    constexpr uint32_t idesc = P16 ? tc::idesc_f16_f16(kTQ, kTN) : tc::idesc_bf16_f32(kTQ, kTN);
    for (int s = 0; s < kSt; ++s) {
        if (s < c.nkt) load_rows<KD, kTN, P16>(tc::smem_addr(c.ring + s * kTile), c.lkp, static_cast<int64_t>(s) * kTN, c.L, c.tid);
        cp_commit();
    }
    for (int t = 0; t <= c.nkt; ++t) {
        if (t >= 1) {
            const uint32_t u = g + t - 1;
            tc::mbar_wait(&c.bars[u & 1], (u >> 1) & 1);
            tc::fence_after_sync();
            const int nxt = t - 1 + kSt;
            if (nxt < c.nkt)
                load_rows<KD, kTN, P16>(tc::smem_addr(c.ring + ((t - 1) % kSt) * kTile), c.lkp,
                                   static_cast<int64_t>(nxt) * kTN, c.L, c.tid);
            cp_commit();
        }
        if (t < c.nkt) {
            cp_wait<kSt - 1>();
            if (P16) cvt_rows_f16<KD, kTN, true>(c.ring + (t % kSt) * kTile, c.tid);
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
            if (P16) {
                uint32_t r0[32];
                tc::ld_32x32b_x32_pack16(base, r0);
                tc::wait_ld();
                f(u, r0, 0);
            } else {
                uint32_t r0[32], r1[32];
                tc::ld_32x32b_x32(base, r0);
                tc::ld_32x32b_x32(base + 32, r1);
                tc::wait_ld();
                f(u, r0, 0);
                f(u, r1, 32);
            }
            tc::fence_before_sync();
        }
        // TMEM buffer (t-1)&1 is next written by MMA(t+1), issued only after
        // the __syncthreads of iteration t+1, which every thread reaches
        // after draining tile t-1 here -- so the only barrier needed per
        // tile is that one; keep one at the end of the pass for the caller
        if (t == c.nkt) __syncthreads();
    }
    cp_wait<0>();
    g += static_cast<uint32_t>(c.nkt);
}

}  // namespace rs
}  // namespace dsa
