// Phase 2: warp-per-row top-k for ROW_TOPK masks with L <= 2048 (C1 and
// every short row-top-k config), per-tensor or per-row scales.
//
// A CTA owns 64 query rows of one pair and stages that pair's K~ levels once
// in shared memory as int8 (exact: |level| <= 127), so a score is four DP4A
// per 16 levels.  One warp per row: each lane holds its NPL = L/32 keys
// (columns lane + 32u) in registers as order-preserving 32-bit rank keys,
// and a warp radix select (8-bit digits, warp-private shared histogram,
// REDUX AND/OR pre-scan skipping common leading bits) finds the keep-th key
// with __syncwarp only -- no CTA barriers per row.
//
// Per-row scales rank by the double product d = s * sk_j; the
// select runs on f = fl32(fl32(s) * fl32(sk_j)), within 2 ulps of d.  Keys
// more than 8 ulps above the threshold are certainly kept, keys more than 8
// ulps below certainly dropped; the few in between are ranked by the exact
// double product (ties: lowest column), as the oracle
// (dsa_oracle_mask_topk_rowscaled) and the reference comparator
// (P/src/linalg.cpp:77-80) do.  Rows whose boundary group exceeds the list
// go to the overflow list finished by the CTA-per-row kernel.
#include <cuda_bf16.h>

#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"

namespace dsa {
namespace {

constexpr int kRW = 8;      // warps per CTA
constexpr int kRowsPerCta = 64;
constexpr int kCand = 256;  // boundary candidates per row

__device__ __forceinline__ uint32_t ord_key(float f) {
    const uint32_t b = __float_as_uint(f == 0.f ? 0.f : f);
    const uint32_t o = (b >> 31) ? ~b : (b | 0x80000000u);  // ascending with f
    return ~o;                                               // smaller = better
}

__device__ __forceinline__ unsigned lane_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

struct RowWarpSmem {
    uint32_t hist[kRW][256];
    uint32_t flags[kRW][64];    // boundary keys taken (bit per column, L <= 2048)
    uint16_t cand[kRW][kCand];  // boundary candidate columns
};

template <int KD, int NPL, bool SCALED>
__global__ void __launch_bounds__(kRW * 32)
    topk_rowwarp_kernel(SelectArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr int kW4 = KD / 4;  // int32 words per level row
    const int L = static_cast<int>(a.L);
    const int Lp = NPL * 32;
    int8_t* kl = reinterpret_cast<int8_t*>(dsm);                        // [Lp][KD]
    float* skf = reinterpret_cast<float*>(dsm + Lp * KD);                // [Lp]
    RowWarpSmem& sw = *reinterpret_cast<RowWarpSmem*>(dsm + Lp * KD + Lp * 4);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t pair = blockIdx.y;
    const uint16_t* lkp = a.lk + pair * a.L * KD;
    const uint16_t* lqp = a.lq + pair * a.L * KD;
    const double* skp = SCALED ? a.sk + pair * a.L : nullptr;

    // stage the pair's K~ levels as int8 (8 levels per 16-byte planar chunk)
    for (int t = tid; t < Lp * (KD / 8); t += kRW * 32) {
        const int r = t / (KD / 8), c = t % (KD / 8);
        uint2 packed = make_uint2(0u, 0u);
        if (r < L) {
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(lkp + lvl_index(a.L, r, c * 8)));
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
            uint32_t b[2] = {0u, 0u};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int lo = static_cast<int>(__uint_as_float(ww[h] << 16));
                const int hi = static_cast<int>(__uint_as_float(ww[h] & 0xffff0000u));
                b[h >> 1] |= ((static_cast<uint32_t>(lo) & 0xffu) | ((static_cast<uint32_t>(hi) & 0xffu) << 8))
                             << ((h & 1) * 16);
            }
            packed = make_uint2(b[0], b[1]);
        }
        *reinterpret_cast<uint2*>(kl + r * KD + c * 8) = packed;
    }
    if (SCALED)
        for (int j = tid; j < Lp; j += kRW * 32) skf[j] = j < L ? static_cast<float>(__ldg(skp + j)) : 0.f;
    __syncthreads();

    uint32_t* hist = sw.hist[warp];
    uint32_t* flags = sw.flags[warp];
    uint16_t* cand = sw.cand[warp];
    const uint32_t keep = static_cast<uint32_t>(a.keep);
    const unsigned lt = lane_lt();

    for (int rr = warp; rr < kRowsPerCta; rr += kRW) {
        const int64_t i = static_cast<int64_t>(blockIdx.x) * kRowsPerCta + rr;
        if (i >= L) break;
        // q levels as packed int8
        int qw[kW4];
#pragma unroll
        for (int v = 0; v < KD / 8; ++v) {
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(lqp + lvl_index(a.L, i, v * 8)));
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t b = 0;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint32_t x = ww[2 * h + e];
                    const int lo = static_cast<int>(__uint_as_float(x << 16));
                    const int hi = static_cast<int>(__uint_as_float(x & 0xffff0000u));
                    b |= ((static_cast<uint32_t>(lo) & 0xffu) | ((static_cast<uint32_t>(hi) & 0xffu) << 8)) << (e * 16);
                }
                qw[v * 2 + h] = static_cast<int>(b);
            }
        }
        auto score = [&](int j) -> int {
            const int4* kr = reinterpret_cast<const int4*>(kl + j * KD);
            int s = 0;
#pragma unroll
            for (int v = 0; v < kW4 / 4; ++v) {
                const int4 w = kr[v];
                s = __dp4a(qw[4 * v], w.x, s);
                s = __dp4a(qw[4 * v + 1], w.y, s);
                s = __dp4a(qw[4 * v + 2], w.z, s);
                s = __dp4a(qw[4 * v + 3], w.w, s);
            }
            return s;
        };
        uint32_t r[NPL];
        uint32_t aa = 0xffffffffu, oo = 0u;
#pragma unroll
        for (int u = 0; u < NPL; ++u) {
            const int j = u * 32 + lane;
            const int s = score(j);
            r[u] = j < L ? ord_key(SCALED ? static_cast<float>(s) * skf[j] : static_cast<float>(s)) : 0xffffffffu;
            if (j < L) {
                aa &= r[u];
                oo |= r[u];
            }
        }
        aa = __reduce_and_sync(0xffffffffu, aa);
        oo = __reduce_or_sync(0xffffffffu, oo);
        // ---- warp radix select: T = keep-th smallest rank key, rem = ties taken
        const uint32_t diff = aa ^ oo;
        uint32_t prefix = aa, rem = keep;
        for (int shift = diff ? ((31 - __clz(diff)) / 8) * 8 : -8; shift >= 0; shift -= 8) {
#pragma unroll
            for (int b = lane; b < 256; b += 32) hist[b] = 0u;
            __syncwarp();
            const uint32_t hm = shift + 8 >= 32 ? 0u : (0xffffffffu << (shift + 8));
#pragma unroll
            for (int u = 0; u < NPL; ++u)
                if (u * 32 + lane < L && (r[u] & hm) == (prefix & hm)) atomicAdd(&hist[(r[u] >> shift) & 255u], 1u);
            __syncwarp();
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                c[e] = hist[lane * 8 + e];
                tot += c[e];
            }
            uint32_t incl = tot;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            const uint32_t excl = incl - tot;
            const bool mine = excl < rem && rem <= incl;
            const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
            uint32_t dsel = 0, newrem = 0;
            if (mine) {
                uint32_t cum = excl;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    if (newrem == 0 && cum + c[e] >= rem) {
                        dsel = static_cast<uint32_t>(lane * 8 + e);
                        newrem = rem - cum;
                    }
                    cum += c[e];
                }
            }
            dsel = __shfl_sync(0xffffffffu, dsel, src);
            rem = __shfl_sync(0xffffffffu, newrem, src);
            prefix = (prefix & ~(0xffu << shift)) | (dsel << shift);
            __syncwarp();
        }
        const uint32_t T = prefix;
        uint32_t* out = a.cols + (pair * a.L + i) * a.keep;
        bool ovf = false;
        if (SCALED) {
            // boundary group: |r - T| <= 8 ulps; certainly kept: r < T - 8
            const uint32_t lo = T >= 8u ? T - 8u : 0u, hi = T <= 0xfffffff7u ? T + 8u : 0xffffffffu;
            uint32_t na = 0, nb = 0;
#pragma unroll
            for (int b = lane; b < 64; b += 32) flags[b] = 0u;
            __syncwarp();
#pragma unroll
            for (int u = 0; u < NPL; ++u) {
                const int j = u * 32 + lane;
                const bool in_a = j < L && r[u] < lo;
                const bool in_b = j < L && r[u] >= lo && r[u] <= hi;
                na += __popc(__ballot_sync(0xffffffffu, in_a));
                const unsigned bb = __ballot_sync(0xffffffffu, in_b);
                const uint32_t pos = nb + __popc(bb & lt);
                if (in_b && pos < kCand) cand[pos] = static_cast<uint16_t>(j);
                nb += __popc(bb);
            }
            __syncwarp();
            if (nb > kCand) {
                ovf = true;
            } else {
                const uint32_t need = keep - na;  // from the boundary group
                for (uint32_t c = lane; c < nb; c += 32) {
                    const int j = cand[c];
                    const double d = static_cast<double>(score(j)) * __ldg(skp + j);
                    uint32_t rank = 0;
                    for (uint32_t c2 = 0; c2 < nb; ++c2) {
                        const int j2 = cand[c2];
                        const double d2 = static_cast<double>(score(j2)) * __ldg(skp + j2);
                        rank += (d2 > d || (d2 == d && j2 < j)) ? 1u : 0u;
                    }
                    if (rank < need) atomicOr(&flags[j >> 5], 1u << (j & 31));
                }
                __syncwarp();
                uint32_t base = 0;
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const int j = u * 32 + lane;
                    const bool take = j < L && (r[u] < lo || (r[u] <= hi && ((flags[u] >> lane) & 1u)));
                    const unsigned bt = __ballot_sync(0xffffffffu, take);
                    if (take) out[base + __popc(bt & lt)] = static_cast<uint32_t>(j);
                    base += __popc(bt);
                }
            }
        } else {
            // exact integer keys: r < T, then the first `rem` equal to T by column
            uint32_t base = 0, eq_seen = 0;
#pragma unroll
            for (int u = 0; u < NPL; ++u) {
                const int j = u * 32 + lane;
                const bool eq = j < L && r[u] == T;
                const unsigned be = __ballot_sync(0xffffffffu, eq);
                const bool take = (j < L && r[u] < T) || (eq && eq_seen + __popc(be & lt) < rem);
                const unsigned bt = __ballot_sync(0xffffffffu, take);
                if (take) out[base + __popc(bt & lt)] = static_cast<uint32_t>(j);
                base += __popc(bt);
                eq_seen += __popc(be);
            }
        }
        if (ovf && lane == 0) {
            const unsigned slot = atomicAdd(a.ovf_n, 1u);
            a.ovf_list[slot] = pair * a.L + i;
        }
        __syncwarp();
    }
}

template <int KD, int NPL>
void launch_rowwarp(const SelectArgs& a, cudaStream_t st) {
    const size_t smem = static_cast<size_t>(NPL * 32) * (KD + 4) + sizeof(RowWarpSmem);
    const dim3 grid(static_cast<unsigned>(ceil_div_i(a.L, kRowsPerCta)), static_cast<unsigned>(a.pairs));
    if (a.per_row) {
        auto kern = topk_rowwarp_kernel<KD, NPL, true>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<grid, kRW * 32, smem, st>>>(a);
    } else {
        auto kern = topk_rowwarp_kernel<KD, NPL, false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<grid, kRW * 32, smem, st>>>(a);
    }
    note_launch();
}

template <int KD>
void dispatch_rowwarp(const SelectArgs& a, cudaStream_t st) {
    if (a.L <= 512) launch_rowwarp<KD, 16>(a, st);
    else if (a.L <= 1024) launch_rowwarp<KD, 32>(a, st);
    else launch_rowwarp<KD, 64>(a, st);
}

}  // namespace

bool topk_rowwarp_supported(const SelectArgs& a) {
    if (a.mode != kRowTopk || (a.KD != 16 && a.KD != 32) || a.L > 2048) return false;
    // opt-in (DSA_TOPK_WARP=1): parity-tested, but measured slower than the
    // CTA-per-row radix kernel (C1 3.25 vs 3.07 ms, C0 0.054 vs 0.013 ms):
    // the first radix digits of clustered keys serialise the warp-private
    // histogram atomics, and 248 registers leave one CTA per SM
    if (std::getenv("DSA_TOPK_WARP") == nullptr) return false;
    // per-row scales need the overflow list; exact int8 levels (|level| <= 127)
    return (!a.per_row || a.ovf_n != nullptr) && a.qmax <= 127;
}

void run_topk_rowwarp(const SelectArgs& a, cudaStream_t st) {
    if (a.per_row) cudaMemsetAsync(a.ovf_n, 0, sizeof(unsigned), st);
    if (a.KD == 16) dispatch_rowwarp<16>(a, st);
    else dispatch_rowwarp<32>(a, st);
    if (a.per_row) launch_topk_scaled_list(a, a.ovf_list, a.ovf_n, st);  // overflow rows (normally none)
}

}  // namespace dsa
