// Phase 2 fast path for vector-wise masks (COLVEC, v = 8): tcgen05 score
// GEMM fused with band max-pooling and exact top-k selection.
//
// One CTA owns 128 query rows (16 bands of 8) of one (b,h) pair and streams
// every key tile of 128 keys through the 5th-gen tensor core:
//
//   D[key, q] = sum_c K~[key, c] * Q~[q, c]      tcgen05.mma kind::f16,
//                                                 M = 128 keys, N = 128 queries,
//                                                 K = 16 (one instruction per tile)
//
// Levels are small integers held exactly in bf16 and the fp32 accumulator
// is exact (|S| < 2^24), so D is the exact integer score S^T.
// D is double-buffered in TMEM (2 x 128 columns) so the MMA of tile t
// overlaps the epilogue of tile t-1.  In the epilogue every thread owns one
// TMEM lane = one key and reads its 128 query columns (tcgen05.ld 32x32b);
// the band max over 8 consecutive columns is in-register (FMNMX3), so
// max-pooling needs no shuffles.  Pooled scores stay in shared memory
// (int16) and each warp then selects its bands with an exact histogram
// select (value desc, lowest index first among equals, P/src/linalg.cpp:
// 77-80), emitting the ascending column list.  The L x L score matrix never
// exists in HBM.
#include <cuda_bf16.h>


#include "device_common.cuh"
#include "kernels.h"
#include "band_core.cuh"
#include "select_common.cuh"
#include "tc_sm100.cuh"

namespace dsa {
namespace {

using namespace sel;

constexpr int kMT = 128;      // keys per tile (UMMA M)
constexpr int kStages = 6;    // K~ tile ring
constexpr int kAcc = 4;       // TMEM accumulators (tiles in flight between MMA and epilogue)
constexpr int kLag = 2;       // MMA issue runs kLag tiles ahead of the epilogue
constexpr int kThreads = 256;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }


// Canonical K-major no-swizzle layout for a [rows][KD] bf16 tile:
// 8-row x 16-byte core matrices, K-adjacent cores 128 B apart (LBO),
// row groups KD*16 B apart (SBO).
template <int KD>
__device__ __forceinline__ uint32_t tile_off(int r, int chunk16) {
    return static_cast<uint32_t>((r >> 3) * (KD * 16) + chunk16 * 128 + (r & 7) * 16);
}

template <int KD, int ROWS = kMT, int NT = kThreads>
__device__ __forceinline__ void load_tile(uint32_t sbase, const uint16_t* __restrict__ src,
                                          int64_t row0, int64_t L, int tid) {
    constexpr int kCh = KD / 8;  // 16-byte chunks per row
    for (int t = tid; t < ROWS * kCh; t += NT) {
        const int r = t / kCh, c = t % kCh;
        const bool ok = row0 + r < L;
        cp_async16(sbase + tile_off<KD>(r, c), src + lvl_index(L, ok ? (row0 + r) : 0, c * 8), ok);
    }
}

template <int KD>
struct ColvecSmem {
    static constexpr int kTileBytes = kMT * KD * 2;
};

// NQ = 64: 8 bands per CTA, ~100 KB of shared memory -> two CTAs per SM, so
// one CTA's selection overlaps the other's tensor-core / TMEM score loop.
// (A TMA-engine variant of the K~ tile copies -- one bulk copy per 8-column
// plane, per-slot mbarriers -- measured slower on C2: 0.85 vs 0.70 ms.)

// Fused select + attention (FUSED, NQ = 64, d = 64): after its bands are
// selected, each warp runs the band attention (band_core.cuh) over its
// band's list straight from shared memory -- the mask never touches HBM
// (`out` may be NULL) and one CTA's memory-bound gathers overlap the other
// resident CTA's ALU-bound score loop / selection.
struct FusedAttn {
    const __nv_bfloat16* q;
    const __nv_bfloat16* k;
    const __nv_bfloat16* v;
    __nv_bfloat16* z;
    int scale;
};

// threads per CTA: four warps per 32-query column group (TMEM lane quarters)
template <int NQ>
constexpr int colvec_threads() { return NQ == 32 ? 128 : 256; }

constexpr int kTPS = 2;                 // key tiles per pipeline step (one barrier per step)
constexpr int kSS = kStages / kTPS;     // step slots in the K~ ring
constexpr int kAS = kAcc / kTPS;        // TMEM accumulator sets

template <int KD, int NQ, bool FUSED = false>
__global__ void __launch_bounds__(colvec_threads<NQ>(), NQ == 128 ? 1 : (NQ == 64 ? 2 : 4))
    colvec_tc_kernel(const uint16_t* __restrict__ lq, const uint16_t* __restrict__ lk, int64_t L,
                     int64_t keep, int M, uint32_t* __restrict__ out, FusedAttn fa) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int kT = colvec_threads<NQ>();
    constexpr int NB = NQ / 8;       // bands per CTA
    constexpr int CPW = NQ / (kT / 128);  // query columns per epilogue warp (lane quarter x column group)
    constexpr int NLD = CPW / 32;    // tcgen05.ld x32 per tile
    constexpr int BPW = CPW / 8;     // bands per warp
    constexpr int kTile = ColvecSmem<KD>::kTileBytes;
    const int Li = static_cast<int>(L);
    const int nt = (Li + kMT - 1) / kMT;
    const int Lp = nt * kMT;
    unsigned char* p = smem;
    unsigned char* bq = p;                      p += NQ * KD * 2;         // Q~ block (N = NQ)
    unsigned char* ring = p;                    p += kStages * kTile;     // K~ tiles
    int16_t* pooled = reinterpret_cast<int16_t*>(p); p += NB * Lp * 2;   // [band][key]
    uint32_t* hist = reinterpret_cast<uint32_t*>(p); p += (kT / 32) * 64 * 4;
    uint32_t* obufs = reinterpret_cast<uint32_t*>(p); p += (kT / 32) * kList * 4;
    int* bandmax = reinterpret_cast<int*>(p);   p += 16 * 4;
    uint64_t* bars = reinterpret_cast<uint64_t*>(p);  // one per TMEM accumulator set
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kAcc + kStages + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int quarter = warp & 3, half = warp >> 2;  // TMEM lane quarter, column half
    const int64_t pair = blockIdx.y;
    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * NQ;
    const uint16_t* lqp = lq + pair * L * KD;
    const uint16_t* lkp = lk + pair * L * KD;

    if (tid == 0) {
        for (int b = 0; b < kAS; ++b) tc::mbar_init(&bars[b], 1);
        tc::fence_barrier_init();
    }
    if (tid < NB) bandmax[tid] = INT32_MIN;
    if (warp == 0) tc::tmem_alloc<kAcc * NQ>(tmem_slot);

    // each thread copies the same 16-byte chunk(s) of every K~ tile: the
    // chunk-planar levels put tile n's copy of a chunk n * kMT rows further
    // along the same plane, so the per-tile address math is one add
    constexpr int kCPT = kMT * (KD / 8) / kT;  // chunks per thread per tile
    uint32_t soff[kCPT];
    const uint16_t* gsrc[kCPT];
    int rrow[kCPT];
#pragma unroll
    for (int i = 0; i < kCPT; ++i) {
        const int t = tid + i * kT, r = t / (KD / 8), c = t % (KD / 8);
        soff[i] = tile_off<KD>(r, c);
        gsrc[i] = lkp + lvl_index(L, r, c * 8);
        rrow[i] = r;
    }
    const uint32_t ring_s = tc::smem_addr(ring);
    auto load_k = [&](int slot, int tile) {  // tile -> ring slot (tile index)
        const int row0 = tile * kMT;
#pragma unroll
        for (int i = 0; i < kCPT; ++i) {
            const bool ok = row0 + rrow[i] < Li;
            cp_async16(ring_s + slot * kTile + soff[i], gsrc[i] + (ok ? row0 * 8 : 0), ok);
        }
    };
    auto load_step = [&](int sslot, int step) {
#pragma unroll
        for (int i = 0; i < kTPS; ++i)
            if (step * kTPS + i < nt) load_k(sslot * kTPS + i, step * kTPS + i);
    };
    const int ns = (nt + kTPS - 1) / kTPS;  // pipeline steps
    // prologue: Q~ block + first kSS steps (group s <-> step s)
    load_tile<KD, NQ, kT>(tc::smem_addr(bq), lqp, q0, L, tid);
    for (int s = 0; s < kSS; ++s) {
        if (s < ns) load_step(s, s);
        cp_commit();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = tc::idesc_bf16_f32(kMT, NQ);
    const uint64_t bdesc = tc::desc_kmajor_nosw(tc::smem_addr(bq), 128, KD * 16);
    const uint32_t bars_s = tc::smem_addr(bars);
    const bool ragged_q = q0 + NQ > L;
    float bmax[BPW];
#pragma unroll
    for (int i = 0; i < BPW; ++i) bmax[i] = -INFINITY;
    const uint32_t tlane = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + half * CPW;

    // Software pipeline over steps of kTPS key tiles: iteration t issues the
    // MMAs of step t (accumulator set t % kAS) and drains step t - 1, whose
    // MMAs finished during the previous epilogue; its ring slot is then
    // refilled with step t - 1 + kSS.  One __syncthreads per step.  Step j's
    // copies are commit group j (j < kSS) or j + 1, so when step t is needed
    // at most kSS - 2 younger groups may still be in flight.
    for (int t = 0; t < ns + 1; ++t) {
        if (t < ns) {
            cp_wait<kSS - 2>();
            tc::fence_proxy_async();
        }
        __syncthreads();
        if (t < ns && tid == 0) {
            tc::fence_after_sync();
#pragma unroll
            for (int i = 0; i < kTPS; ++i) {
                if (t * kTPS + i >= nt) break;
                const uint32_t abase = ring_s + ((t % kSS) * kTPS + i) * kTile;
#pragma unroll
                for (int ks = 0; ks < KD / 16; ++ks) {
                    const uint64_t ad = tc::desc_kmajor_nosw(abase + ks * 256, 128, KD * 16);
                    const uint64_t bd = bdesc + static_cast<uint64_t>((ks * 256) >> 4);
                    tc::mma_bf16(tmem + ((t % kAS) * kTPS + i) * NQ, ad, bd, idesc, ks > 0);
                }
            }
            tc::commit_a(bars_s + (t % kAS) * 8);
        }
        if (t >= 1) {
            const int u = t - 1;
            tc::mbar_wait_a(bars_s + (u % kAS) * 8, (u / kAS) & 1);
            tc::fence_after_sync();
#pragma unroll
            for (int i = 0; i < kTPS; ++i) {
                const int tile = u * kTPS + i;
                if (tile >= nt) break;
                // epilogue of one tile: thread = key tile*128 + 32*quarter + lane,
                // query columns [CPW*half, CPW*half + CPW)
                const int key = tile * kMT + quarter * 32 + lane;
                const bool kvalid = key < Li;
                const uint32_t base = tlane + ((u % kAS) * kTPS + i) * NQ;
                uint32_t rr[NLD][32];
#pragma unroll
                for (int l = 0; l < NLD; ++l) tc::ld_32x32b_x32(base + l * 32, rr[l]);
                tc::wait_ld();
#pragma unroll
                for (int cb = 0; cb < NLD; ++cb) {
                    uint32_t* r = rr[cb];
                    if (ragged_q) {
#pragma unroll
                        for (int x = 0; x < 32; ++x)
                            if (q0 + half * CPW + cb * 32 + x >= L) r[x] = __float_as_uint(-INFINITY);
                    }
                    float m4[4];
#pragma unroll
                    for (int bb = 0; bb < 4; ++bb) {
                        float m0, m1, m2;
                        const float* f = reinterpret_cast<const float*>(&r[bb * 8]);
                        asm("max.f32 %0, %1, %2, %3;" : "=f"(m0) : "f"(f[0]), "f"(f[1]), "f"(f[2]));
                        asm("max.f32 %0, %1, %2, %3;" : "=f"(m1) : "f"(f[3]), "f"(f[4]), "f"(f[5]));
                        asm("max.f32 %0, %1, %2, %3;" : "=f"(m2) : "f"(m0), "f"(m1), "f"(f[6]));
                        m4[bb] = fmaxf(m2, f[7]);
                        if (kvalid) bmax[cb * 4 + bb] = fmaxf(bmax[cb * 4 + bb], m4[bb]);
                    }
                    // two bands per 32-bit store: [band / 2][key][2] int16 (the
                    // exact integer maxima convert by the 1.5 * 2^23 addition)
#pragma unroll
                    for (int pp = 0; pp < 2; ++pp) {
                        const int v0 = __float_as_int(m4[2 * pp] + 12582912.0f) - 0x4B400000;
                        const int v1 = __float_as_int(m4[2 * pp + 1] + 12582912.0f) - 0x4B400000;
                        const uint32_t packed = kvalid ? __byte_perm(static_cast<uint32_t>(v0), static_cast<uint32_t>(v1), 0x5410)
                                                       : 0x80008000u;
                        const int band = half * BPW + cb * 4 + 2 * pp;  // even
                        *reinterpret_cast<uint32_t*>(pooled + ((band >> 1) * Lp + key) * 2) = packed;
                    }
                }
            }
            tc::fence_before_sync();
            // step u's ring slot is free (its MMAs completed): refill it
            if (u + kSS < ns) load_step(u % kSS, u + kSS);
        }
        cp_commit();
    }
    __syncthreads();
    // band maxima: warp reduce, then shared atomics across the 4 lane quarters
#pragma unroll
    for (int i = 0; i < BPW; ++i) {
        float v = bmax[i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (lane == 0) atomicMax(&bandmax[half * BPW + i], __float2int_rn(v));
    }
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<kAcc * NQ>(tmem);

    // ---- exact per-band selection (one warp per band)
    const int64_t nb = (L + 7) / 8;
    uint32_t* h = hist + warp * 64;
    for (int b = warp; b < NB; b += kT / 32) {
        const int64_t band = q0 / 8 + b;
        if (band >= nb) break;
        const int16_t* pv = pooled + (b >> 1) * Lp * 2 + (b & 1);
        band_select<2>(pv, static_cast<int>(L), Lp, static_cast<int>(keep), bandmax[b], M, h,
                       obufs + warp * kList, out ? out + (pair * nb + band) * keep : nullptr, lane);
        __syncwarp();
    }
    if constexpr (FUSED) {
        static_assert(NQ == 64 && kT / 32 == 8, "fused path: one band per warp");
        // the score-loop buffers (ring, pooled, histograms) are free now
        __syncthreads();
        using BS = bc::BandSmemV2<64>;
        BS& sm = reinterpret_cast<BS*>(ring)[warp];
        const int64_t band = q0 / 8 + warp;
        if (band < nb) {
            const uint32_t* lst = obufs + warp * kList;
            auto chunk_idx = [&](int ch) -> uint32_t {
                const int64_t pidx = static_cast<int64_t>(ch) * 32 + lane;
                return pidx < keep ? lst[pidx] : 0u;
            };
            bc::band_core<64, 8, false>(sm, fa.q, fa.k + pair * L * 64, fa.v + pair * L * 64, pair, L, band * 8,
                                        keep, 0, 0, 0, fa.scale, fa.z, chunk_idx, lane);
        }
    }
}

template <int KD, int NQ>
size_t colvec_smem_bytes(int64_t L) {
    const int64_t nt = (L + kMT - 1) / kMT;
    return ColvecSmem<KD>::kTileBytes * kStages + NQ * KD * 2 + (NQ / 8) * nt * kMT * 2 +
           (colvec_threads<NQ>() / 32) * 64 * 4 + (colvec_threads<NQ>() / 32) * kList * 4 + 16 * 4 +
           (2 * kAcc + kStages + 1) * 8 + 8;
}

}  // namespace

bool colvec_tc_supported(const SelectArgs& a) {
    if (a.mode != kColvec || a.vec_v != 8 || a.per_row || a.qmax > 7) return false;
    if (a.KD != 16 && a.KD != 32) return false;
    if (a.keep > kList - 32) return false;
    const size_t smem = a.KD == 16 ? colvec_smem_bytes<16, 128>(a.L) : colvec_smem_bytes<32, 128>(a.L);
    return smem <= 227 * 1024;
}

template <int KD, int NQ>
void launch_colvec(const SelectArgs& a, int M, cudaStream_t st) {
    const size_t smem = colvec_smem_bytes<KD, NQ>(a.L);
    auto kern = colvec_tc_kernel<KD, NQ, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const dim3 grid(static_cast<unsigned>(ceil_div_i(a.L, NQ)), static_cast<unsigned>(a.pairs));
    kern<<<grid, colvec_threads<NQ>(), smem, st>>>(a.lq, a.lk, a.L, a.keep, M, a.cols, FusedAttn{});
}

void run_colvec_tc(const SelectArgs& a, cudaStream_t st) {
    const int M = static_cast<int>(a.KD) * a.qmax * a.qmax;
    // two 64-query CTAs per SM when their shared memory fits, else one 128-query CTA
    const bool two = (a.KD == 16 ? colvec_smem_bytes<16, 64>(a.L) : colvec_smem_bytes<32, 64>(a.L)) <= 113 * 1024;
    if (a.KD == 16) {
        if (two) launch_colvec<16, 64>(a, M, st);
        else launch_colvec<16, 128>(a, M, st);
    } else {
        if (two) launch_colvec<32, 64>(a, M, st);
        else launch_colvec<32, 128>(a, M, st);
    }
    note_launch();
}

bool colvec_fused_supported(const SelectArgs& s, const AttnArgs& a) {
    if (options().no_fuse) return false;
    if (!colvec_tc_supported(s) || s.KD != 16 || !a.bf16 || a.D != 64 || a.vec_v != 8) return false;
    if (s.keep > kList - 32) return false;  // band list must stay in the staging buffer
    const size_t smem = colvec_smem_bytes<16, 64>(s.L);
    // the per-warp attention buffers reuse the ring + pooled + histogram region
    const size_t reuse = static_cast<size_t>(ColvecSmem<16>::kTileBytes) * kStages +
                         static_cast<size_t>(8) * ((s.L + kMT - 1) / kMT) * kMT * 2 + (kThreads / 32) * 64 * 4;
    return smem <= 113 * 1024 && reuse >= sizeof(bc::BandSmemV2<64>) * 8;
}

void run_colvec_fused(const SelectArgs& s, const AttnArgs& a, cudaStream_t st) {
    const int M = static_cast<int>(s.KD) * s.qmax * s.qmax;
    const size_t smem = colvec_smem_bytes<16, 64>(s.L);
    auto kern = colvec_tc_kernel<16, 64, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const dim3 grid(static_cast<unsigned>(ceil_div_i(s.L, 64)), static_cast<unsigned>(s.pairs));
    FusedAttn fa{static_cast<const __nv_bfloat16*>(a.q), static_cast<const __nv_bfloat16*>(a.k),
                 static_cast<const __nv_bfloat16*>(a.v), static_cast<__nv_bfloat16*>(a.z), a.scale};
    kern<<<grid, kThreads, smem, st>>>(s.lq, s.lk, s.L, s.keep, M, s.cols, fa);
    note_launch();
}

}  // namespace dsa
