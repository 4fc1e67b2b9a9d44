// Phase 2 for vector-wise masks (COLVEC, v = 8, <= 4-bit levels): the exact
// integer score GEMM on the 5th-gen tensor cores fused with band
// max-pooling, an in-flight histogram per band and exact top-k selection,
// optionally fused with the band attention (dsa_pipeline).
//
// Reference rule (P/src/maskgen.cpp:33-61): bands of 8 query
// rows, band score of key j = max over the band rows of the exact integer
// S~[i][j], keep `keep` keys per band by row_topk_indices (value desc, the
// LOWER key first among equals, P/src/linalg.cpp:77-80), ascending list.
//
// One CTA = 64 queries (8 bands) of one (b,h) pair, 10 warps:
//   * warp 8 (TMA producer, one lane): per accumulator slot, its two K~ tiles
//     (256 keys) by ONE bulk copy per 8-column plane straight from the
//     chunk-planar levels into the slot's stage, refilled as soon as the
//     slot's MMAs completed;
//   * warp 9 (MMA issuer, one lane): per slot two tcgen05.mma (M = 128 keys,
//     N = 64 queries, K = 16 per instruction) and ONE commit, which both
//     hands the slot to the epilogue and frees its stage.  (A commit or a
//     bulk copy costs a single issuing thread hundreds of cycles once the SM
//     is busy -- tools/mma_issue_bench.cu, tools/tma_issue_bench.cu -- so a
//     commit per tile plus one per slot capped the score loop: 0.415 ms ->
//     0.371 ms on C2 with one per slot);
//   * warps 0-7 (epilogue): warp w drains TMEM lanes 32 (w & 3).. (= keys)
//     x columns 32 (w >> 2).. (= 4 bands) with ONE tcgen05.ld per tile and
//     frees the accumulator, then per band: max over 8 columns (FMNMX3), one
//     FADD with 1.5 2^23 + 2^14 (bits = 0x4B404000 + v), whose low 16 bits
//     are stored as the band's pooled code (0x4000 + v: a positive normal
//     f16, monotone in v) and whose bits address the band's histogram word
//     (M - v) of one RED -- 8 instructions per (band, key);
// then per band (one warp each): the keep-th largest value T from the
// histogram (top-down cumulative counts, 256 bins per warp step), one pass
// over the band's pooled codes with packed f16 compares (HSET2, 8 keys per
// 16-byte load) building a key bitmap of v >= T, a warp prefix sum placing
// every such key in ascending order, and a pass over that short list
// dropping the surplus ties (lowest keys kept).  The L x L scores never
// leave the SM.
//
// FUSED (d = 64, k = 16): the 8 warps then run the band attention
// (band_core.cuh) on their lists straight from shared memory, so the mask
// never touches HBM unless the caller asks for it.
#include <algorithm>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "band_core.cuh"
#include "device_common.cuh"
#include "kernels.h"
#include "tc_sm100.cuh"

// DSA_ABLATE: profiling builds only (tools/ablate.py; bit 1 -- no selection,
// bit 2 -- no pooling / histogram / codes, bit 32 -- half the key tiles); 0 in
// the library
#ifndef DSA_ABLATE
#define DSA_ABLATE 0
#endif

namespace dsa {
namespace {

constexpr int kMT = 128;       // keys per tile (UMMA M)
constexpr int kNQ = 64;        // queries per CTA (UMMA N) = 8 bands
constexpr int kBands = kNQ / 8;
constexpr int kAcc = 2;        // TMEM accumulator slots, two key tiles (2 kNQ columns) each
constexpr int kEpiWarps = 8;
constexpr int kLoadWarp = kEpiWarps;      // TMA producer
constexpr int kMmaWarp = kEpiWarps + 1;   // tcgen05.mma issuer
constexpr int kThreads = (kEpiWarps + 2) * 32;
constexpr int kList = 512;     // per-band staging list (keys)
constexpr uint32_t kCodeBias = 0x4B404000u;  // bits of 1.5 * 2^23 + 2^14
constexpr float kCodeMagic = 12599296.0f;    // 1.5 * 2^23 + 2^14

template <int KD>
struct Layout {
    static constexpr int kPlanesA = KD / 8;
    static constexpr int kTile = kMT * KD * 2;          // one K~ tile (bytes)
    static constexpr int kStage = 2 * kTile;            // one accumulator slot's two tiles
    static constexpr int kQ = kNQ * KD * 2;             // the Q~ block
    static constexpr int kMaxM = KD * 49;               // |score| bound, qmax <= 7
    static constexpr int kBins = (2 * kMaxM + 1 + 255) / 256 * 256;  // per band pair (u32 = 2 x u16)
    static constexpr int kHist = (kBands / 2) * kBins * 4;
    static constexpr int kObuf = kBands * kList * 4;
    static constexpr int kHistRegion = kHist > kObuf ? kHist : kObuf;
    static constexpr int kBars = (3 * kAcc + 1) * 8 + 16;
    // ring + pooled codes (reused by the fused attention's per-warp buffers)
    __host__ __device__ static size_t work_bytes(int64_t L, bool fused) {
        const size_t nt = static_cast<size_t>((L + kMT - 1) / kMT);
        const size_t w = static_cast<size_t>(kAcc) * kStage + ((DSA_ABLATE & 2) ? 0 : static_cast<size_t>(kBands) * nt * kMT * 2);
        const size_t f = fused ? sizeof(bc::BandSmemV2<64>) * kEpiWarps : 0;
        return w > f ? w : f;
    }
    __host__ __device__ static size_t smem_bytes(int64_t L, bool fused) { return kQ + work_bytes(L, fused) + kHistRegion + kBars; }
};

__device__ __forceinline__ void named_sync_epi() { asm volatile("bar.sync 1, %0;\n" ::"n"(kEpiWarps * 32) : "memory"); }

__device__ __forceinline__ void sts_u16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;\n" ::"r"(addr), "h"(static_cast<unsigned short>(v)) : "memory");
}
__device__ __forceinline__ void red_add(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
    return r;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];\n" : "=h"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint32_t hge2(uint32_t a, uint32_t b) {
    return __hge2_mask(*reinterpret_cast<const __half2*>(&a), *reinterpret_cast<const __half2*>(&b));
}

// Byte offset of key j's pooled code inside its band row (a row = Lp codes):
// 128-key segments of 16 16-byte chunks, chunk c stored at c ^ (seg & 7), so
// 32 lanes reading chunk c of 32 consecutive segments hit every bank group
// 4 times (the minimum), and the epilogue's 32 consecutive keys stay in one
// 128-byte row.
__device__ __forceinline__ uint32_t code_off(int j) {
    const int seg = j >> 7, c = (j >> 3) & 15;
    return static_cast<uint32_t>(((seg << 4) + (c ^ (seg & 7))) << 4) + ((j & 7) << 1);
}

// The keep-th largest pooled value T of one band and the counts above / at
// it, from the band's histogram (bins v = M .. -M at word offsets 0 ..;
// 16-bit half `sh` of each u32 word; W * 32 words).  One warp, two scans:
// lane l sums its W consecutive bins (a band's counts fit 16 bits, so the
// other band's half never carries into this one), a warp prefix sum finds
// the lane whose range holds the keep-th value, then that range's bins are
// spread over the warp (W / 32 rounded up per lane) and scanned again.
struct BandCut {
    int T = 0;
    uint32_t n_gt = 0, n_eq = 0;
};
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}
template <int W>
__device__ __forceinline__ BandCut band_cut(uint32_t hp, int sh, int M, int keep, int lane) {
    static_assert(W % 4 == 0, "16-byte histogram reads");
    constexpr int kPer = W <= 64 ? 2 : 4;  // bins per lane in the second scan
    static_assert(W <= 32 * kPer, "second scan covers the range");
    uint32_t acc = 0;
    const uint32_t base = hp + static_cast<uint32_t>(lane * W * 4);
#pragma unroll
    for (int i = 0; i < W; i += 4) {
        const uint4 x = lds128(base + i * 4);
        acc += x.x + x.y + x.z + x.w;
    }
    const uint32_t mine = (acc >> sh) & 0xFFFFu;
    const uint32_t incl = warp_incl_scan(mine, lane);
    const unsigned hit = __ballot_sync(0xffffffffu, incl >= static_cast<uint32_t>(keep));
    const int f = hit ? __ffs(hit) - 1 : 31;
    const uint32_t carry = __shfl_sync(0xffffffffu, incl - mine, f);
    // the W bins of lane f, kPer per lane
    const int b0 = f * W + kPer * lane;
    uint32_t c[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) c[i] = 0;
    if (kPer * lane < W) {
        if constexpr (kPer == 2) {
            uint32_t x, y;
            asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];\n" : "=r"(x), "=r"(y) : "r"(hp + b0 * 4));
            c[0] = (x >> sh) & 0xFFFFu;
            c[1] = (y >> sh) & 0xFFFFu;
        } else {
            const uint4 x = lds128(hp + b0 * 4);
            c[0] = (x.x >> sh) & 0xFFFFu;
            c[1] = (x.y >> sh) & 0xFFFFu;
            c[2] = (x.z >> sh) & 0xFFFFu;
            c[3] = (x.w >> sh) & 0xFFFFu;
        }
    }
    uint32_t m2 = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) m2 += c[i];
    const uint32_t incl2 = warp_incl_scan(m2, lane);
    const unsigned hit2 = __ballot_sync(0xffffffffu, carry + incl2 >= static_cast<uint32_t>(keep));
    const int f2 = hit2 ? __ffs(hit2) - 1 : 31;
    int tt = 0;
    uint32_t gt = 0, eq = 0;
    if (lane == f2) {
        uint32_t run = carry + incl2 - m2;
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            if (run + c[i] >= static_cast<uint32_t>(keep)) {
                tt = M - (b0 + i);
                gt = run;
                eq = c[i];
                break;
            }
            run += c[i];
        }
    }
    BandCut r;
    r.T = __shfl_sync(0xffffffffu, tt, f2);
    r.n_gt = __shfl_sync(0xffffffffu, gt, f2);
    r.n_eq = __shfl_sync(0xffffffffu, eq, f2);
    return r;
}

// The band's ascending list of kept keys (value desc, lowest key first among
// equals at T) from its pooled codes `prow_s`, in ONE pass: per 128-key
// segment (one per lane) packed f16 compares build bitmaps of v > T and
// v >= T, a warp prefix sum over the tie counts admits the first `rem` ties
// (lowest keys first), a second prefix sum over the kept counts places each
// lane's keys in the staging list `obuf` (keep entries, ascending); then the
// list is copied to `o` when given.  One warp.
__device__ __forceinline__ void band_emit(const BandCut& cut, uint32_t prow_s, uint32_t* obuf, uint32_t* o, int keep,
                                          int Lp, int lane) {
    const uint32_t codeT = 0x4000u + static_cast<uint32_t>(cut.T);
    const uint32_t rem = static_cast<uint32_t>(keep) - cut.n_gt;  // ties admitted, lowest keys first
    const int nseg = Lp / kMT;
    const uint32_t T2 = codeT | (codeT << 16), U2 = (codeT + 1u) | ((codeT + 1u) << 16);
    uint32_t eq_base = 0, k_base = 0;
    for (int s0 = 0; s0 < nseg; s0 += 32) {
        const int seg = s0 + lane;
        uint32_t wg[4] = {0u, 0u, 0u, 0u}, we[4] = {0u, 0u, 0u, 0u};  // v > T, v >= T
        if (seg < nseg) {
            const uint32_t sb = prow_s + static_cast<uint32_t>(seg) * 256;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const uint4 x = lds128(sb + static_cast<uint32_t>((c ^ (seg & 7)) << 4));
                uint32_t te = hge2(x.x, T2) & 0x00020001u, tg = hge2(x.x, U2) & 0x00020001u;
                te |= hge2(x.y, T2) & 0x00080004u;
                tg |= hge2(x.y, U2) & 0x00080004u;
                te |= hge2(x.z, T2) & 0x00200010u;
                tg |= hge2(x.z, U2) & 0x00200010u;
                te |= hge2(x.w, T2) & 0x00800040u;
                tg |= hge2(x.w, U2) & 0x00800040u;
                we[c >> 2] |= ((te | (te >> 16)) & 0xFFu) << ((c & 3) * 8);
                wg[c >> 2] |= ((tg | (tg >> 16)) & 0xFFu) << ((c & 3) * 8);
            }
        }
        // ties: admit this lane's first (rem - ties before it) tie keys
        uint32_t ne = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) ne += __popc(we[j] & ~wg[j]);
        const uint32_t eincl = warp_incl_scan(ne, lane);
        const uint32_t ebefore = eq_base + eincl - ne;
        uint32_t allow = rem > ebefore ? rem - ebefore : 0u;
        uint32_t nk = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t eqj = we[j] & ~wg[j];
            const uint32_t cj = __popc(eqj);
            if (allow < cj) {
                // keep the first `allow` ties of this word: bits below the (allow+1)-th set bit
                eqj = allow == 0 ? 0u : eqj & ((1u << __fns(eqj, 0, allow + 1)) - 1u);
                allow = 0;
            } else {
                allow -= cj;
            }
            we[j] = wg[j] | eqj;
            nk += __popc(we[j]);
        }
        const uint32_t kincl = warp_incl_scan(nk, lane);
        uint32_t pos = k_base + kincl - nk;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t x = we[j];
            while (x) {
                const int bit = __ffs(x) - 1;
                x &= x - 1;
                obuf[pos++] = static_cast<uint32_t>(seg * kMT + j * 32 + bit);
            }
        }
        eq_base += __shfl_sync(0xffffffffu, eincl, 31);
        k_base += __shfl_sync(0xffffffffu, kincl, 31);
    }
    __syncwarp();
    if (o)
        for (int i = lane; i < keep; i += 32) o[i] = obuf[i];
    __syncwarp();
}

struct FusedAttn {
    const __nv_bfloat16* q;
    const __nv_bfloat16* k;
    const __nv_bfloat16* v;
    __nv_bfloat16* z;
    int scale;
};

template <int KD, bool FUSED>
__global__ void __launch_bounds__(kThreads, 2)
    colvec_kernel(const uint16_t* __restrict__ lq, const uint16_t* __restrict__ lk, int L, int keep, int M,
                  uint32_t* __restrict__ out, FusedAttn fa) {
    using Lay = Layout<KD>;
    extern __shared__ __align__(1024) unsigned char smem[];
    const int Lp = (L + kMT - 1) / kMT * kMT;
    const int nt = (DSA_ABLATE & 32) ? Lp / kMT / 2 : Lp / kMT;  // profiling: half the key tiles
    const size_t work = Lay::work_bytes(L, FUSED);
    unsigned char* q_sm = smem;
    unsigned char* ring = smem + Lay::kQ;
    unsigned char* pooled = ring + kAcc * Lay::kStage;
    unsigned char* histp = smem + Lay::kQ + work;
    uint64_t* bars = reinterpret_cast<uint64_t*>(histp + Lay::kHistRegion);
    uint64_t* full = bars;                   // [kAcc] a slot's stage landed (TMA -> MMA)
    uint64_t* accf = bars + kAcc;            // [kAcc] MMAs of a slot done -> epilogue, stage free
    uint64_t* acce = accf + kAcc;            // [kAcc] slot drained -> MMA (8 arrivals)
    uint64_t* qbar = acce + kAcc;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qbar + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t pair = blockIdx.y;
    const int q0 = blockIdx.x * kNQ;
    const uint16_t* lqp = lq + pair * static_cast<int64_t>(L) * KD;
    const uint16_t* lkp = lk + pair * static_cast<int64_t>(L) * KD;

    if (tid == 0) {
        for (int i = 0; i < kAcc; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&accf[i], 1);
            tc::mbar_init(&acce[i], kEpiWarps);
        }
        tc::mbar_init(qbar, 1);
        tc::fence_barrier_init();
    }
    {  // zero the band histograms
        uint4* h4 = reinterpret_cast<uint4*>(histp);
        for (int i = tid; i < Lay::kHist / 16; i += kThreads) h4[i] = make_uint4(0, 0, 0, 0);
    }
    if (warp == 0) tc::tmem_alloc<kAcc * 2 * kNQ>(tmem_slot);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp == kLoadWarp) {
        // ------------------------------------------------- TMA producer
        if (lane == 0) {
            const uint32_t ring_s = tc::smem_addr(ring), q_s = tc::smem_addr(q_sm);
            {
                const int rows = L - q0 < kNQ ? L - q0 : kNQ;
                tc::mbar_expect_tx(qbar, static_cast<uint32_t>(rows * 16 * Lay::kPlanesA));
#pragma unroll
                for (int c = 0; c < Lay::kPlanesA; ++c)
                    tc::bulk_g2s(q_s + c * (kNQ * 16), lqp + (static_cast<int64_t>(c) * L + q0) * 8,
                                 static_cast<uint32_t>(rows * 16), qbar);
            }
            // one stage per accumulator slot (two key tiles, [plane][256 keys][16 B]:
            // ONE bulk copy per plane), refilled once the slot's MMAs completed
            for (int u = 0; 2 * u < nt; ++u) {
                const int a = u % kAcc;
                if (u >= kAcc) tc::mbar_wait_susp(&accf[a], ((u / kAcc) - 1) & 1);
                const int row0 = 2 * u * kMT;
                const int rows = L - row0 < 2 * kMT ? L - row0 : 2 * kMT;
                tc::mbar_expect_tx(&full[a], static_cast<uint32_t>(rows * 16 * Lay::kPlanesA));
#pragma unroll
                for (int c = 0; c < Lay::kPlanesA; ++c)
                    tc::bulk_g2s(ring_s + a * Lay::kStage + c * (2 * kMT * 16),
                                 lkp + (static_cast<int64_t>(c) * L + row0) * 8, static_cast<uint32_t>(rows * 16),
                                 &full[a]);
            }
        }
        return;
    }
    if (warp == kMmaWarp) {
        // ------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t ring_s = tc::smem_addr(ring), q_s = tc::smem_addr(q_sm);
            const uint32_t idesc = tc::idesc_bf16_f32(kMT, kNQ);
            tc::mbar_wait(qbar, 0);
            // per slot: two key tiles, ONE commit (it frees the stage and hands the
            // slot to the epilogue) -- a commit costs the issuing thread hundreds
            // of cycles (tools/mma_issue_bench.cu), a commit per tile capped the loop
            for (int u = 0; 2 * u < nt; ++u) {
                const int a = u % kAcc;
                if (u >= kAcc) tc::mbar_wait_susp(&acce[a], ((u / kAcc) - 1) & 1);
                tc::mbar_wait_susp(&full[a], (u / kAcc) & 1);
                tc::fence_after_sync();
                for (int i = 0; i < 2 && 2 * u + i < nt; ++i) {
#pragma unroll
                    for (int ks = 0; ks < KD / 16; ++ks) {
                        // K-major, no swizzle: 8-row x 16-byte core matrices; the
                        // two K-adjacent ones are the two 8-column planes
                        // (LBO = the stage's plane stride), 8-row groups 128 B apart (SBO)
                        const uint64_t ad = tc::desc_kmajor_nosw(
                            ring_s + a * Lay::kStage + i * (kMT * 16) + ks * 2 * (2 * kMT * 16), 2 * kMT * 16, 128);
                        const uint64_t bd = tc::desc_kmajor_nosw(q_s + ks * 2 * (kNQ * 16), kNQ * 16, 128);
                        tc::mma_bf16(tmem + (2 * a + i) * kNQ, ad, bd, idesc, ks > 0);
                    }
                }
                tc::commit(&accf[a]);
            }
        }
        return;
    }

    // ---------------------------------------------------------- epilogue
    const int quarter = warp & 3, half = warp >> 2;
    const uint32_t tl = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + half * 32;
    const uint32_t pooled_s = tc::smem_addr(pooled);
    const uint32_t hist_s = tc::smem_addr(histp);
    const uint32_t row_bytes = static_cast<uint32_t>(Lp) * 2;
    // histogram word of band b, value v: pair (b / 2), index M - v; the code
    // bits are kCodeBias + v, so the address is one IMAD: C_b - 4 code
    uint32_t hc[4], inc[4], prow[4];
    bool bvalid[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int band = half * 4 + b;
        hc[b] = hist_s + static_cast<uint32_t>((band >> 1) * Lay::kBins * 4) + 4u * static_cast<uint32_t>(M) + 4u * kCodeBias;
        inc[b] = (band & 1) ? 0x10000u : 1u;
        prow[b] = pooled_s + static_cast<uint32_t>(band) * row_bytes;
        bvalid[b] = q0 + band * 8 < L;
    }
    const bool ragged_q = q0 + kNQ > L;
    const int cbase = quarter * 4 + (lane >> 3);  // this thread's 16-byte chunk in a 128-key segment
    const uint32_t ebyte = static_cast<uint32_t>(lane & 7) << 1;

    // per tile: 4 bands x (max of 8 columns, code, pooled store, histogram RED)
    auto process = [&](int t, const uint32_t (&r)[32]) {
        const uint32_t off = (static_cast<uint32_t>((t << 4) + (cbase ^ (t & 7))) << 4) + ebyte;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const float* f = reinterpret_cast<const float*>(&r[b * 8]);
            float m0, m1, m2;
            asm("max.f32 %0, %1, %2, %3;" : "=f"(m0) : "f"(f[0]), "f"(f[1]), "f"(f[2]));
            asm("max.f32 %0, %1, %2, %3;" : "=f"(m1) : "f"(f[3]), "f"(f[4]), "f"(f[5]));
            asm("max.f32 %0, %1, %2, %3;" : "=f"(m2) : "f"(m0), "f"(m1), "f"(f[6]));
            const uint32_t code = __float_as_uint(fmaxf(m2, f[7]) + kCodeMagic);
            sts_u16(prow[b] + off, code);
            red_add(hc[b] - 4u * code, inc[b]);
        }
    };
    // the same with ragged keys (last tile) / ragged queries (last CTA of a pair)
    auto process_edge = [&](int t, uint32_t (&r)[32]) {
        const int key = t * kMT + quarter * 32 + lane;
        const uint32_t off = (static_cast<uint32_t>((t << 4) + (cbase ^ (t & 7))) << 4) + ebyte;
#pragma unroll
        for (int x = 0; x < 32; ++x)
            if (q0 + half * 32 + x >= L) r[x] = __float_as_uint(-INFINITY);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const float* f = reinterpret_cast<const float*>(&r[b * 8]);
            float m = f[0];
#pragma unroll
            for (int x = 1; x < 8; ++x) m = fmaxf(m, f[x]);
            const uint32_t code = __float_as_uint(m + kCodeMagic);
            const bool ok = key < L && bvalid[b];
            sts_u16(prow[b] + off, ok ? code : 0u);  // 0: below every valid code
            if (ok) red_add(hc[b] - 4u * code, inc[b]);
        }
    };
    const int edge_from = ragged_q ? 0 : (Lp != L ? nt - 1 : nt);  // first tile needing the edge path

    for (int u = 0; 2 * u < nt; ++u) {
        const int a = u % kAcc;
        tc::mbar_wait_susp(&accf[a], (u / kAcc) & 1);
        tc::fence_after_sync();
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int t = 2 * u + i;
            if (t >= nt) break;
            uint32_t r[32];
            tc::ld_32x32b_x32(tl + (2 * a + i) * kNQ, r);
            tc::wait_ld();
            if (i == 1 || t + 1 == nt) {  // slot drained
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&acce[a]);
            }
            if (DSA_ABLATE & 2) { if (r[0] == 0x7fffffffu) red_add(hist_s, r[1]); continue; }  // profiling build only
            if (t < edge_from) process(t, r);
            else process_edge(t, r);
        }
    }
    named_sync_epi();  // every score drained, every code and count in place
    if (warp == 0) tc::tmem_dealloc<kAcc * 2 * kNQ>(tmem);
    if (DSA_ABLATE & 1) return;  // profiling build only: no selection

    // ------------------------------------------------ per-band selection
    const int band = q0 / 8 + warp;  // this warp's band (global index within the pair)
    const int nbands = (L + 7) / 8;
    const bool live = band < nbands;
#if DSA_ABLATE & 128  // profiling build only: selection phase cycles (CTA 0, warp 0)
    const long long c0 = clock64();
#endif
    const BandCut cut = live ? band_cut<Lay::kBins / 32>(hist_s + static_cast<uint32_t>((warp >> 1) * Lay::kBins * 4),
                                                         (warp & 1) * 16, M, keep, lane)
                             : BandCut{};
#if DSA_ABLATE & 128
    const long long c1 = clock64();
#endif
    named_sync_epi();  // histograms consumed: the staging lists reuse them
#if DSA_ABLATE & 128
    const long long c2 = clock64();
#endif
    uint32_t* obuf = reinterpret_cast<uint32_t*>(histp) + warp * kList;
    if (live)
        band_emit(cut, pooled_s + static_cast<uint32_t>(warp) * row_bytes, obuf,
                  out ? out + (pair * nbands + band) * static_cast<int64_t>(keep) : nullptr, keep, Lp, lane);
#if DSA_ABLATE & 128
    if ((blockIdx.x == 5 && blockIdx.y == 3) && lane == 0)
        printf("warp %d cut %lld sync %lld emit %lld T %d ngt %u neq %u\n", warp, c1 - c0, c2 - c1, clock64() - c2, cut.T, cut.n_gt, cut.n_eq);
#endif
    if constexpr (FUSED) {
        named_sync_epi();  // ring + pooled codes free: per-warp attention buffers
        using BS = bc::BandSmemV2<64>;
        BS& sm = reinterpret_cast<BS*>(ring)[warp];
        if (live) {
            auto chunk_idx = [&](int ch) -> uint32_t {
                const int p = ch * 32 + lane;
                return p < keep ? obuf[p] : 0u;
            };
            bc::band_core<64, 8, false>(sm, fa.q, fa.k + pair * static_cast<int64_t>(L) * 64,
                                        fa.v + pair * static_cast<int64_t>(L) * 64, pair, L,
                                        static_cast<int64_t>(band) * 8, keep, 0, 0, 0, fa.scale, fa.z, chunk_idx,
                                        lane);
        }
    }
}

template <int KD, bool FUSED>
void launch(const SelectArgs& s, const FusedAttn& fa, cudaStream_t st) {
    const size_t smem = Layout<KD>::smem_bytes(s.L, FUSED);
    auto kern = colvec_kernel<KD, FUSED>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const dim3 grid(static_cast<unsigned>(ceil_div_i(s.L, kNQ)), static_cast<unsigned>(s.pairs));
    const int M = static_cast<int>(s.KD) * s.qmax * s.qmax;
    kern<<<grid, kThreads, smem, st>>>(s.lq, s.lk, static_cast<int>(s.L), static_cast<int>(s.keep), M, s.cols, fa);
    note_launch();
}

}  // namespace

bool colvec_tc_supported(const SelectArgs& a) {
    if (a.mode != kColvec || a.vec_v != 8 || a.per_row || a.qmax > 7) return false;
    if (a.KD != 16 && a.KD != 32) return false;
    if (a.keep > kList - 32) return false;
    const size_t smem = a.KD == 16 ? Layout<16>::smem_bytes(a.L, false) : Layout<32>::smem_bytes(a.L, false);
    return smem <= 227 * 1024;
}

void run_colvec_tc(const SelectArgs& a, cudaStream_t st) {
    if (a.KD == 16) launch<16, false>(a, FusedAttn{}, st);
    else launch<32, false>(a, FusedAttn{}, st);
}

bool colvec_fused_supported(const SelectArgs& s, const AttnArgs& a) {
    if (!options().fuse) return false;
    if (!colvec_tc_supported(s) || s.KD != 16 || !a.bf16 || a.D != 64 || a.vec_v != 8) return false;
    return Layout<16>::smem_bytes(s.L, true) <= 227 * 1024;
}

void run_colvec_fused(const SelectArgs& s, const AttnArgs& a, cudaStream_t st) {
    const FusedAttn fa{static_cast<const __nv_bfloat16*>(a.q), static_cast<const __nv_bfloat16*>(a.k),
                       static_cast<const __nv_bfloat16*>(a.v), static_cast<__nv_bfloat16*>(a.z), a.scale};
    launch<16, true>(s, fa, st);
}

}  // namespace dsa
