// Exact per-band top-k selection helpers shared by the tensor-core select
// kernels: windowed histogram / binary-search threshold and the ascending
// ballot emission (value desc, lowest column first among ties,
// P/src/linalg.cpp:77-80).
#pragma once

#include <stdint.h>

namespace dsa {
namespace sel {

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

constexpr int kWin = 512;  // histogram scratch per warp (bins)

// Counts values >= lo into h[0..W) and returns the count inside the window.
// S: element stride of the pooled values (1: one band per row; 2: two bands
// interleaved as int16 pairs)
template <int W, int S = 1>
__device__ __forceinline__ uint32_t window_hist(const int16_t* __restrict__ pv, int L, int lo,
                                                uint32_t* h, int lane) {
    for (int i = lane; i < W; i += 32) h[i] = 0;
    __syncwarp();
    // branch-free: the bin address is v * 4 + (h - 4 lo), the reduction is
    // predicated on v >= lo (no divergent branch around each atomic)
    const uint32_t hb = static_cast<uint32_t>(__cvta_generic_to_shared(h)) - static_cast<uint32_t>(lo) * 4u;
    auto add = [&](int v) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ge.s32 p, %1, %2;\n\t@p red.shared.add.u32 [%0], 1;\n\t}\n" ::"r"(
                         hb + static_cast<uint32_t>(v) * 4u),
                     "r"(v), "r"(lo)
                     : "memory");
    };
    int j = lane;
    for (; j + 96 < L; j += 128) {
        const int v0 = pv[j * S], v1 = pv[(j + 32) * S], v2 = pv[(j + 64) * S], v3 = pv[(j + 96) * S];
        add(v0);
        add(v1);
        add(v2);
        add(v3);
    }
    for (; j < L; j += 32) add(pv[j * S]);
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
                                                 int& T, uint32_t& rem, uint32_t& nT) {
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
    uint32_t r = 0, n = 0;
    if (mine) {
        uint32_t cum = excl;
#pragma unroll
        for (int i = per - 1; i >= 0; --i) {
            if (r == 0 && cum + c[i] >= kk) {
                t = lo + lane * per + i;
                r = kk - cum;
                n = c[i];
            }
            cum += c[i];
        }
    }
    T = __shfl_sync(0xffffffffu, t, src);
    rem = __shfl_sync(0xffffffffu, r, src);
    nT = __shfl_sync(0xffffffffu, n, src);
}

// Exact selection of one band from pooled[0..L) (int16 scores): threshold T
// = keep-th largest value, rem = how many values == T to admit (lowest
// column first).  The keep-th largest sits a few dozen below the band max,
// so counting starts on a 64-value window (few shared atomics), widens to
// 512, and falls back to a binary search over the full integer range.
// nge = count(v >= T) when known from the histogram, else UINT32_MAX.
template <int S = 1>
__device__ __forceinline__ void band_threshold(const int16_t* __restrict__ pv, int L, int keep,
                                               int bmax, int M, uint32_t* h, int lane, int& T,
                                               uint32_t& rem, uint32_t& nge) {
    const uint32_t kk = static_cast<uint32_t>(keep);
    nge = 0xffffffffu;
    if (window_hist<64, S>(pv, L, bmax - 63, h, lane) >= kk) {
        uint32_t nT;
        window_threshold<64>(h, bmax - 63, kk, lane, T, rem, nT);
        nge = kk - rem + nT;
        return;
    }
    const int lo = bmax - 63;
    // rare: keep-th value below the window -> binary search on count(v >= x)
    int a = -M, b = lo - 1;  // invariant: count(v >= a) >= keep, count(v >= b + 1) < keep
    while (a < b) {
        const int mid = a + (b - a + 1) / 2;
        uint32_t cnt = 0;
        for (int jj = lane; jj < L; jj += 32) cnt += pv[jj * S] >= mid;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        if (cnt >= kk) a = mid;
        else b = mid - 1;
    }
    T = a;
    uint32_t above = 0;
    for (int jj = lane; jj < L; jj += 32) above += pv[jj * S] > T;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) above += __shfl_xor_sync(0xffffffffu, above, off);
    rem = kk - above;
}

// Ascending emission: every column with value > T, then values == T in
// column order until `rem` of them are taken.
template <int S = 1>
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
            v[u] = j < L ? pv[j * S] : INT32_MIN;
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

constexpr int kList = 512;  // per-band output staging (column indices)

__device__ __forceinline__ unsigned vote_ballot(bool p) {
    unsigned r;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tvote.sync.ballot.b32 %0, q, 0xffffffff;\n\t}\n"
                 : "=r"(r)
                 : "r"(static_cast<unsigned>(p)));
    return r;
}

// Exact top-`keep` of one band (pooled[0..Lp), padded columns INT16_MIN):
// threshold from the windowed histogram, then one ascending pass that
// stages every column with value >= T in shared memory (one ballot per 32
// columns), a short pass over that list dropping the ties beyond `rem`
// (lowest columns first), and the copy of the list to global memory.  When
// the >= T set does not fit the staging list, the two-ballot emission with
// a trash slot is used instead.  The final list is left in obuf[0, keep)
// (for a fused consumer); o may be NULL (no global copy).
template <int S = 1>
__device__ __forceinline__ void band_select(const int16_t* __restrict__ pv, int L, int Lp, int keep,
                                            int bmax, int M, uint32_t* h, uint32_t* obuf,
                                            uint32_t* __restrict__ o, int lane) {
    int T;
    uint32_t rem, nge;
    band_threshold<S>(pv, L, keep, bmax, M, h, lane, T, rem, nge);
    if (keep > kList - 32) {
        band_emit<S>(pv, L, keep, T, rem, o, lane);
        return;
    }
    const unsigned lt = lanemask_lt();
    if (nge <= static_cast<uint32_t>(kList)) {
        uint32_t taken = 0;
        const uint32_t ob = static_cast<uint32_t>(__cvta_generic_to_shared(obuf));
        for (int j0 = 0; j0 < Lp; j0 += 128) {
            int v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = pv[(j0 + u * 32 + lane) * S];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool ge = v[u] >= T;
                const unsigned b = vote_ballot(ge);
                // predicated store: no divergent branch per value
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ge.s32 p, %2, %3;\n\t@p st.shared.u32 [%0], %1;\n\t}\n" ::"r"(
                                 ob + (taken + __popc(b & lt)) * 4u),
                             "r"(static_cast<uint32_t>(j0 + u * 32 + lane)), "r"(v[u]), "r"(T)
                             : "memory");
                taken += __popc(b);
            }
        }
        __syncwarp();
        if (nge == static_cast<uint32_t>(keep)) {
            if (o)
                for (int i = lane; i < keep; i += 32) o[i] = obuf[i];
        } else {  // admit only the first `rem` columns equal to T (compacted in place)
            uint32_t eq_seen = 0, outp = 0;
            for (uint32_t i0 = 0; i0 < nge; i0 += 32) {
                const uint32_t i = i0 + lane;
                const bool valid = i < nge;
                const uint32_t col = valid ? obuf[i] : 0u;
                const bool eq = valid && pv[col * S] == T;
                const unsigned be = vote_ballot(eq);
                const bool kp = valid && (!eq || eq_seen + __popc(be & lt) < rem);
                const unsigned bk = vote_ballot(kp);
                __syncwarp();  // every lane read its entry before any write below
                if (kp) {
                    obuf[outp + __popc(bk & lt)] = col;
                    if (o) o[outp + __popc(bk & lt)] = col;
                }
                outp += __popc(bk);
                eq_seen += __popc(be);
            }
        }
        __syncwarp();
        return;
    }
    const uint32_t trash = static_cast<uint32_t>(kList - 32 + lane);
    uint32_t taken = 0, eq_seen = 0;
    for (int j0 = 0; j0 < Lp; j0 += 128) {
        int v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = pv[(j0 + u * 32 + lane) * S];
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
    if (o)
        for (int i = lane; i < keep; i += 32) o[i] = obuf[i];
    __syncwarp();
}


}  // namespace sel
}  // namespace dsa
