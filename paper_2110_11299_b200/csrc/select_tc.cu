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

#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"
#include "tc_sm100.cuh"

namespace dsa {
namespace {

constexpr int kNQ = 128;      // queries per CTA (16 bands)
constexpr int kMT = 128;      // keys per tile (UMMA M)
constexpr int kStages = 4;    // K~ tile ring
constexpr int kThreads = 256;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Canonical K-major no-swizzle layout for a [rows][KD] bf16 tile:
// 8-row x 16-byte core matrices, K-adjacent cores 128 B apart (LBO),
// row groups KD*16 B apart (SBO).
template <int KD>
__device__ __forceinline__ uint32_t tile_off(int r, int chunk16) {
    return static_cast<uint32_t>((r >> 3) * (KD * 16) + chunk16 * 128 + (r & 7) * 16);
}

template <int KD>
__device__ __forceinline__ void load_tile(uint32_t sbase, const uint16_t* __restrict__ src,
                                          int64_t row0, int64_t L, int tid) {
    constexpr int kCh = KD / 8;  // 16-byte chunks per row
    for (int t = tid; t < kMT * kCh; t += kThreads) {
        const int r = t / kCh, c = t % kCh;
        const bool ok = row0 + r < L;
        cp_async16(sbase + tile_off<KD>(r, c), src + (ok ? (row0 + r) : 0) * KD + c * 8, ok);
    }
}

template <int KD>
struct ColvecSmem {
    static constexpr int kTileBytes = kMT * KD * 2;
};

constexpr int kWin = 512;  // histogram scratch per warp (bins)

// Counts values >= lo into h[0..W) and returns the count inside the window.
template <int W>
__device__ __forceinline__ uint32_t window_hist(const int16_t* __restrict__ pv, int L, int lo,
                                                uint32_t* h, int lane) {
    for (int i = lane; i < W; i += 32) h[i] = 0;
    __syncwarp();
    int j = lane;
    for (; j + 96 < L; j += 128) {
        const int v0 = pv[j], v1 = pv[j + 32], v2 = pv[j + 64], v3 = pv[j + 96];
        if (v0 >= lo) atomicAdd(&h[v0 - lo], 1u);
        if (v1 >= lo) atomicAdd(&h[v1 - lo], 1u);
        if (v2 >= lo) atomicAdd(&h[v2 - lo], 1u);
        if (v3 >= lo) atomicAdd(&h[v3 - lo], 1u);
    }
    for (; j < L; j += 32) {
        const int v = pv[j];
        if (v >= lo) atomicAdd(&h[v - lo], 1u);
    }
    __syncwarp();
    uint32_t c = 0;
    for (int i = lane; i < W; i += 32) c += h[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    return c;
}

// T = the keep-th largest value (bins are values lo..lo+W-1), rem = number
// of values == T admitted.  Requires count(window) >= keep.
template <int W>
__device__ __forceinline__ void window_threshold(const uint32_t* h, int lo, uint32_t kk, int lane,
                                                 int& T, uint32_t& rem) {
    constexpr int per = W / 32;
    uint32_t c[per], local = 0;
#pragma unroll
    for (int i = 0; i < per; ++i) {
        c[i] = h[lane * per + i];
        local += c[i];
    }
    uint32_t suf = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, suf, off);
        if (lane + off < 32) suf += y;
    }
    const uint32_t excl = suf - local;
    const bool mine = excl < kk && kk <= suf;
    const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
    int t = 0;
    uint32_t r = 0;
    if (mine) {
        uint32_t cum = excl;
#pragma unroll
        for (int i = per - 1; i >= 0; --i) {
            if (r == 0 && cum + c[i] >= kk) {
                t = lo + lane * per + i;
                r = kk - cum;
            }
            cum += c[i];
        }
    }
    T = __shfl_sync(0xffffffffu, t, src);
    rem = __shfl_sync(0xffffffffu, r, src);
}

// Exact selection of one band from pooled[0..L) (int16 scores): threshold T
// = keep-th largest value, rem = how many values == T to admit (lowest
// column first).  The keep-th largest sits a few dozen below the band max,
// so counting starts on a 64-value window (few shared atomics), widens to
// 512, and falls back to a binary search over the full integer range.
__device__ __forceinline__ void band_threshold(const int16_t* __restrict__ pv, int L, int keep,
                                               int bmax, int M, uint32_t* h, int lane, int& T,
                                               uint32_t& rem) {
    const uint32_t kk = static_cast<uint32_t>(keep);
    if (window_hist<64>(pv, L, bmax - 63, h, lane) >= kk) {
        window_threshold<64>(h, bmax - 63, kk, lane, T, rem);
        return;
    }
    const int lo = bmax - (kWin - 1);
    if (window_hist<kWin>(pv, L, lo, h, lane) >= kk) {
        window_threshold<kWin>(h, lo, kk, lane, T, rem);
        return;
    }
    // rare: keep-th value below the window -> binary search on count(v >= x)
    int a = -M, b = lo - 1;  // invariant: count(v >= a) >= keep, count(v >= b + 1) < keep
    while (a < b) {
        const int mid = a + (b - a + 1) / 2;
        uint32_t cnt = 0;
        for (int jj = lane; jj < L; jj += 32) cnt += pv[jj] >= mid;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        if (cnt >= kk) a = mid;
        else b = mid - 1;
    }
    T = a;
    uint32_t above = 0;
    for (int jj = lane; jj < L; jj += 32) above += pv[jj] > T;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) above += __shfl_xor_sync(0xffffffffu, above, off);
    rem = kk - above;
}

// Ascending emission: every column with value > T, then values == T in
// column order until `rem` of them are taken.
__device__ __forceinline__ void band_emit(const int16_t* __restrict__ pv, int L, int keep, int T,
                                          uint32_t rem, uint32_t* __restrict__ o, int lane) {
    const uint32_t kk = static_cast<uint32_t>(keep);
    const unsigned lt = lanemask_lt();
    uint32_t taken = 0, eq_seen = 0;
    for (int j0 = 0; j0 < L && taken < kk; j0 += 128) {
        int v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = j0 + u * 32 + lane;
            v[u] = j < L ? pv[j] : INT32_MIN;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool gt = v[u] > T, eq = v[u] == T;
            const unsigned be = __ballot_sync(0xffffffffu, eq);
            const bool take = gt || (eq && eq_seen + __popc(be & lt) < rem);
            const unsigned bt = __ballot_sync(0xffffffffu, take);
            if (take) o[taken + __popc(bt & lt)] = static_cast<uint32_t>(j0 + u * 32 + lane);
            taken += __popc(bt);
            eq_seen += __popc(be);
        }
    }
}

constexpr int kList = 1024;  // per-warp output staging (column indices)

__device__ __forceinline__ unsigned vote_ballot(bool p) {
    unsigned r;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tvote.sync.ballot.b32 %0, q, 0xffffffff;\n\t}\n"
                 : "=r"(r)
                 : "r"(static_cast<unsigned>(p)));
    return r;
}

// Exact top-`keep` of one band (pooled[0..Lp), padded columns INT16_MIN):
// threshold from the windowed histogram, then one ascending pass that
// stages kept columns in shared memory (unconditional stores; dropped lanes
// write a trash slot) and a coalesced copy of the list to global memory.
__device__ __forceinline__ void band_select(const int16_t* __restrict__ pv, int L, int Lp, int keep,
                                            int bmax, int M, uint32_t* h, uint32_t* obuf,
                                            uint32_t* __restrict__ o, int lane) {
    int T;
    uint32_t rem;
    band_threshold(pv, L, keep, bmax, M, h, lane, T, rem);
    if (keep > kList - 32) {
        band_emit(pv, L, keep, T, rem, o, lane);
        return;
    }
    const unsigned lt = lanemask_lt();
    const uint32_t trash = static_cast<uint32_t>(kList - 32 + lane);
    uint32_t taken = 0, eq_seen = 0;
    for (int j0 = 0; j0 < Lp; j0 += 128) {
        int v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = pv[j0 + u * 32 + lane];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool eq = v[u] == T;
            const unsigned be = vote_ballot(eq);
            const bool take = v[u] > T || (eq && eq_seen + __popc(be & lt) < rem);
            const unsigned bt = vote_ballot(take);
            obuf[take ? taken + __popc(bt & lt) : trash] = static_cast<uint32_t>(j0 + u * 32 + lane);
            taken += __popc(bt);
            eq_seen += __popc(be);
        }
    }
    __syncwarp();
    for (int i = lane; i < keep; i += 32) o[i] = obuf[i];
    __syncwarp();
}

template <int KD>
__global__ void __launch_bounds__(kThreads, 1)
    colvec_tc_kernel(const uint16_t* __restrict__ lq, const uint16_t* __restrict__ lk, int64_t L,
                     int64_t keep, int M, uint32_t* __restrict__ out, int dbg) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int kTile = ColvecSmem<KD>::kTileBytes;
    const int nt = static_cast<int>((L + kMT - 1) / kMT);
    const int Lp = nt * kMT;
    unsigned char* p = smem;
    unsigned char* bq = p;                      p += kTile;               // Q~ block (N = 128)
    unsigned char* ring = p;                    p += kStages * kTile;     // K~ tiles
    int16_t* pooled = reinterpret_cast<int16_t*>(p); p += 16 * Lp * 2;   // [band][key]
    uint32_t* hist = reinterpret_cast<uint32_t*>(p); p += (kThreads / 32) * kWin * 4;
    uint32_t* obufs = reinterpret_cast<uint32_t*>(p); p += (kThreads / 32) * kList * 4;
    int* bandmax = reinterpret_cast<int*>(p);   p += 16 * 4;
    uint64_t* bars = reinterpret_cast<uint64_t*>(p);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int quarter = warp & 3, half = warp >> 2;  // TMEM lane quarter, column half
    const int64_t pair = blockIdx.y;
    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * kNQ;
    const uint16_t* lqp = lq + pair * L * KD;
    const uint16_t* lkp = lk + pair * L * KD;

    if (tid == 0) {
        tc::mbar_init(&bars[0], 1);
        tc::mbar_init(&bars[1], 1);
        tc::fence_barrier_init();
    }
    if (tid < 16) bandmax[tid] = INT32_MIN;
    if (warp == 0) tc::tmem_alloc<256>(tmem_slot);

    // prologue: Q~ block + first kStages K~ tiles (group t <-> tile t)
    load_tile<KD>(tc::smem_addr(bq), lqp, q0, L, tid);
    for (int s = 0; s < kStages; ++s) {
        if (s < nt) load_tile<KD>(tc::smem_addr(ring + s * kTile), lkp, static_cast<int64_t>(s) * kMT, L, tid);
        cp_commit();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = tc::idesc_bf16_f32(kMT, kNQ);
    const uint64_t bdesc = tc::desc_kmajor_nosw(tc::smem_addr(bq), 128, KD * 16);
    const bool ragged_q = q0 + kNQ > L;
    float bmax[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) bmax[i] = -INFINITY;

    for (int t = 0; t <= nt; ++t) {
        if (t >= 1) {
            tc::mbar_wait(&bars[(t - 1) & 1], ((t - 1) >> 1) & 1);
            tc::fence_after_sync();
            const int nxt = t - 1 + kStages;
            if (nxt < nt)
                load_tile<KD>(tc::smem_addr(ring + ((t - 1) % kStages) * kTile), lkp,
                              static_cast<int64_t>(nxt) * kMT, L, tid);
            cp_commit();
        }
        if (t < nt) {
            cp_wait<kStages - 1>();
            tc::fence_proxy_async();
            __syncthreads();
            if (tid == 0) {
                tc::fence_after_sync();
                const uint32_t abase = tc::smem_addr(ring + (t % kStages) * kTile);
#pragma unroll
                for (int ks = 0; ks < KD / 16; ++ks) {
                    const uint64_t ad = tc::desc_kmajor_nosw(abase + ks * 256, 128, KD * 16);
                    const uint64_t bd = bdesc + static_cast<uint64_t>((ks * 256) >> 4);
                    tc::mma_bf16(tmem + (t & 1) * kNQ, ad, bd, idesc, ks > 0);
                }
                tc::commit(&bars[t & 1]);
            }
        }
        if (t >= 1) {
            // epilogue of tile u = t-1: thread = key u*128 + 32*quarter + lane,
            // query columns [64*half, 64*half + 64) = bands 8*half .. 8*half+7
            const int u = t - 1;
            const int key = u * kMT + quarter * 32 + lane;
            const bool kvalid = key < L;
            const uint32_t base = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + (u & 1) * kNQ + half * 64;
            uint32_t r0[32], r1[32];
            tc::ld_32x32b_x32(base, r0);
            tc::ld_32x32b_x32(base + 32, r1);
            tc::wait_ld();
            if (dbg & 2) {  // profiling switch: TMEM reads only
                uint32_t x = 0;
#pragma unroll
                for (int i = 0; i < 32; ++i) x ^= r0[i] ^ r1[i];
                pooled[half * 8 * Lp + key] = static_cast<int16_t>(x);
            } else
#pragma unroll
            for (int cb = 0; cb < 2; ++cb) {
                uint32_t* r = cb ? r1 : r0;
                if (ragged_q) {
#pragma unroll
                    for (int x = 0; x < 32; ++x)
                        if (q0 + half * 64 + cb * 32 + x >= L) r[x] = __float_as_uint(-INFINITY);
                }
#pragma unroll
                for (int bb = 0; bb < 4; ++bb) {
                    float m0, m1, m2;
                    const float* f = reinterpret_cast<const float*>(&r[bb * 8]);
                    asm("max.f32 %0, %1, %2, %3;" : "=f"(m0) : "f"(f[0]), "f"(f[1]), "f"(f[2]));
                    asm("max.f32 %0, %1, %2, %3;" : "=f"(m1) : "f"(f[3]), "f"(f[4]), "f"(f[5]));
                    asm("max.f32 %0, %1, %2, %3;" : "=f"(m2) : "f"(m0), "f"(m1), "f"(f[6]));
                    const float mx = fmaxf(m2, f[7]);
                    const int band = half * 8 + cb * 4 + bb;
                    pooled[band * Lp + key] = kvalid ? static_cast<int16_t>(__float2int_rn(mx)) : INT16_MIN;
                    if (kvalid) bmax[cb * 4 + bb] = fmaxf(bmax[cb * 4 + bb], mx);
                }
            }
            tc::fence_before_sync();
        }
        __syncthreads();
    }
    // band maxima: warp reduce, then shared atomics across the 4 lane quarters
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float v = bmax[i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (lane == 0) atomicMax(&bandmax[half * 8 + i], __float2int_rn(v));
    }
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<256>(tmem);

    // ---- exact per-band selection (one warp per band)
    const int64_t nb = (L + 7) / 8;
    uint32_t* h = hist + warp * kWin;
    for (int b = warp; b < 16 && !(dbg & 1); b += kThreads / 32) {
        const int64_t band = q0 / 8 + b;
        if (band >= nb) break;
        const int16_t* pv = pooled + b * Lp;
        band_select(pv, static_cast<int>(L), Lp, static_cast<int>(keep), bandmax[b], M, h,
                    obufs + warp * kList, out + (pair * nb + band) * keep, lane);
        __syncwarp();
    }
}

template <int KD>
size_t colvec_smem_bytes(int64_t L, int M) {
    const int64_t nt = (L + kMT - 1) / kMT;
    const size_t nbins = static_cast<size_t>(2 * M + 1);
    (void)nbins;
    return ColvecSmem<KD>::kTileBytes * (1 + kStages) + 16 * nt * kMT * 2 +
           (kThreads / 32) * kWin * 4 + (kThreads / 32) * kList * 4 + 16 * 4 + 2 * 8 + 8;
}

}  // namespace

bool colvec_tc_supported(const SelectArgs& a) {
    if (a.mode != kColvec || a.vec_v != 8 || a.per_row || a.qmax > 7) return false;
    if (a.KD != 16 && a.KD != 32) return false;
    const int M = static_cast<int>(a.KD) * a.qmax * a.qmax;
    const size_t smem = a.KD == 16 ? colvec_smem_bytes<16>(a.L, M) : colvec_smem_bytes<32>(a.L, M);
    return smem <= 227 * 1024;
}

void run_colvec_tc(const SelectArgs& a, cudaStream_t st) {
    // DSA_PROFILE_SWITCH: profiling-only ablations (1: skip selection, 2: TMEM reads only)
    static const int dbg = [] {
        const char* e = std::getenv("DSA_PROFILE_SWITCH");
        return e ? std::atoi(e) : 0;
    }();
    const int M = static_cast<int>(a.KD) * a.qmax * a.qmax;
    const dim3 grid(static_cast<unsigned>(ceil_div_i(a.L, kNQ)), static_cast<unsigned>(a.pairs));
    if (a.KD == 16) {
        const size_t smem = colvec_smem_bytes<16>(a.L, M);
        cudaFuncSetAttribute(colvec_tc_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        colvec_tc_kernel<16><<<grid, kThreads, smem, st>>>(a.lq, a.lk, a.L, a.keep, M, a.cols, dbg);
    } else {
        const size_t smem = colvec_smem_bytes<32>(a.L, M);
        cudaFuncSetAttribute(colvec_tc_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        colvec_tc_kernel<32><<<grid, kThreads, smem, st>>>(a.lq, a.lk, a.L, a.keep, M, a.cols, dbg);
    }
    note_launch();
}

}  // namespace dsa
