// Phase 2: exact-integer approximate scores -> mask selection.
//
// Selection semantics are the reference's row_topk_indices comparator
// (value descending, then LOWEST column index; output ascending,
// P/src/linalg.cpp:69-85) applied to the exact integer score
// S[i][j] = <levels_q[i], levels_k[j]>.  Ties are never
// broken by arrival order: a radix select finds the exact k-th key T, every
// key better than T is kept, and keys equal to T are admitted in ascending
// column order (prefix counts) until `keep` is reached.
//
// This file holds the CTA-per-row CUDA-core kernels, used for every mode
// and shape; the tensor-core fast paths (select_tc.cu) take over the
// configurations they are specialised for.
#include <cub/cub.cuh>
#include <climits>
#include <cstdlib>
#include <cuda_bf16.h>

#include "device_common.cuh"
#include "kernels.h"

namespace dsa {
namespace {

constexpr int kNT = 128;
constexpr int kWarps = kNT / 32;

struct SelSmem {
    uint32_t hist[256];
    uint32_t wtot[2][kWarps];
    unsigned long long red[kWarps];
    unsigned long long bcast[4];
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <class KeyT>
__device__ __forceinline__ int key_bits() { return static_cast<int>(sizeof(KeyT) * 8); }

// Block-wide radix select: the keep-th smallest key T (1-based) among
// keys[0..n) and rem = how many keys equal to T belong to the first `keep`.
// Only the digits where keys differ are visited (AND/OR pre-scan).
template <class KeyT>
__device__ void block_radix_select(const KeyT* keys, int n, int keep, SelSmem& s, KeyT& T,
                                   uint32_t& rem) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    KeyT a = ~KeyT(0), o = 0;
    for (int j = tid; j < n; j += kNT) {
        a &= keys[j];
        o |= keys[j];
    }
    // block AND / OR
    unsigned long long aa = a, oo = o;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        aa &= __shfl_xor_sync(0xffffffffu, aa, off);
        oo |= __shfl_xor_sync(0xffffffffu, oo, off);
    }
    if (lane == 0) s.red[warp] = aa;
    __syncthreads();
    if (tid == 0) {
        unsigned long long ta = ~0ull;
        for (int w = 0; w < kWarps; ++w) ta &= s.red[w];
        s.bcast[0] = ta;
    }
    __syncthreads();
    if (lane == 0) s.red[warp] = oo;
    __syncthreads();
    if (tid == 0) {
        unsigned long long to = 0;
        for (int w = 0; w < kWarps; ++w) to |= s.red[w];
        s.bcast[1] = to;
        const unsigned long long diff = (s.bcast[0] ^ to);
        int top = diff ? 63 - __clzll(static_cast<long long>(diff)) : 0;
        s.bcast[2] = static_cast<unsigned long long>(top);
        s.bcast[3] = static_cast<unsigned long long>(keep);
    }
    __syncthreads();
    const unsigned long long common = s.bcast[0];
    const int top = static_cast<int>(s.bcast[2]);
    KeyT prefix = static_cast<KeyT>(common);  // bits above `top` are common to all keys
    uint32_t r = static_cast<uint32_t>(keep);
    int shift = (top / 8) * 8;
    for (; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += kNT) s.hist[i] = 0;
        __syncthreads();
        const KeyT hi_mask = (shift + 8 >= key_bits<KeyT>()) ? KeyT(0) : (~KeyT(0) << (shift + 8));
        for (int j = tid; j < n; j += kNT) {
            const KeyT key = keys[j];
            if ((key & hi_mask) == (prefix & hi_mask))
                atomicAdd(&s.hist[static_cast<uint32_t>(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (warp == 0) {
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                c[u] = s.hist[lane * 8 + u];
                tot += c[u];
            }
            uint32_t incl = tot;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            const uint32_t excl = incl - tot;
            const bool mine = excl < r && r <= incl;
            const unsigned who = __ballot_sync(0xffffffffu, mine);
            if (mine) {
                uint32_t cum = excl;
                int dsel = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (cum + c[u] >= r) {
                        dsel = u;
                        break;
                    }
                    cum += c[u];
                }
                s.bcast[0] = static_cast<unsigned long long>(lane * 8 + dsel);
                s.bcast[1] = static_cast<unsigned long long>(r - cum);
            }
            (void)who;
        }
        __syncthreads();
        const KeyT digit = static_cast<KeyT>(s.bcast[0]);
        r = static_cast<uint32_t>(s.bcast[1]);
        prefix = (prefix & ~(KeyT(255) << shift)) | (digit << shift);
        __syncthreads();
    }
    T = prefix;
    rem = r;
}

// Ordered emission: writes, in ascending index order, every j with
// lt(j), plus the first `rem` (by index) with eq(j).  Returns the count.
template <class Flags>
__device__ uint32_t block_emit(int n, uint32_t rem, Flags flags, uint32_t* out, SelSmem& s) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t base_out = 0, base_eq = 0;
    for (int j0 = 0; j0 < n; j0 += kNT) {
        const int j = j0 + tid;
        bool lt = false, eq = false;
        if (j < n) flags(j, lt, eq);
        const unsigned beq = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) s.wtot[0][warp] = __popc(beq);
        __syncthreads();
        uint32_t eq_off = 0, eq_tot = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t t = s.wtot[0][w];
            eq_off += w < warp ? t : 0;
            eq_tot += t;
        }
        const uint32_t eq_rank = base_eq + eq_off + __popc(beq & lanemask_lt());
        const bool take = lt || (eq && eq_rank < rem);
        const unsigned bt = __ballot_sync(0xffffffffu, take);
        if (lane == 0) s.wtot[1][warp] = __popc(bt);
        __syncthreads();
        uint32_t t_off = 0, t_tot = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t t = s.wtot[1][w];
            t_off += w < warp ? t : 0;
            t_tot += t;
        }
        if (take && out) out[base_out + t_off + __popc(bt & lanemask_lt())] = static_cast<uint32_t>(j);
        base_out += t_tot;
        base_eq += eq_tot;
        __syncthreads();
    }
    return base_out;
}

// row r of one pair's chunk-planar levels ([KD/8][L][8]) as floats
template <int KD>
__device__ __forceinline__ void load_levels(const uint16_t* __restrict__ pairbase, int64_t L, int64_t row,
                                            float (&x)[KD]) {
#pragma unroll
    for (int v = 0; v < KD / 8; ++v) {
        uint4 r = __ldg(reinterpret_cast<const uint4*>(pairbase + lvl_index(L, row, v * 8)));
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            x[v * 8 + 2 * u] = __uint_as_float(w[u] << 16);
            x[v * 8 + 2 * u + 1] = __uint_as_float(w[u] & 0xffff0000u);
        }
    }
}

// Exact: |products| <= 127^2 and |sums| < 2^24, so fp32 FMA is exact.
template <int KD>
__device__ __forceinline__ int score_with(const float (&q)[KD], const uint16_t* __restrict__ kbase, int64_t L,
                                          int64_t j) {
    float kk[KD];
    load_levels<KD>(kbase, L, j, kk);
    float acc = 0.f;
#pragma unroll
    for (int t = 0; t < KD; ++t) acc = fmaf(q[t], kk[t], acc);
    return static_cast<int>(acc);
}

// ---------------------------------------------------------------- top-k
template <class KeyT, int KD>
__global__ void __launch_bounds__(kNT) topk_rows_generic(SelectArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    KeyT* keys = reinterpret_cast<KeyT*>(dsm);
    __shared__ SelSmem s;
    const int64_t i = blockIdx.x, pair = blockIdx.y;
    const int L = static_cast<int>(a.L);
    float q[KD];
    load_levels<KD>(a.lq + pair * a.L * KD, a.L, i, q);
    const uint16_t* lk = a.lk + pair * a.L * KD;
    for (int j = threadIdx.x; j < L; j += kNT) {
        const int sc = score_with<KD>(q, lk, a.L, j);
        if constexpr (sizeof(KeyT) == 8)
            keys[j] = rank_key_f64(static_cast<double>(sc) * a.sk[pair * a.L + j]);
        else
            keys[j] = rank_key_i32(sc);
    }
    __syncthreads();
    KeyT T;
    uint32_t rem;
    block_radix_select<KeyT>(keys, L, static_cast<int>(a.keep), s, T, rem);
    uint32_t* out = a.cols + (pair * a.L + i) * a.keep;
    block_emit(L, rem, [&](int j, bool& lt, bool& eq) {
        lt = keys[j] < T;
        eq = keys[j] == T;
    }, out, s);
}

// row_topk_indices on ANY f64 matrix (P/src/linalg.cpp:69-85): the rule the
// masks above apply to S~, for callers that rank scores of their own -- the
// reference's oracle_topk_mask(Q K^T, keep) (P/src/maskgen.cpp:11-16) is this
// on the exact scores.  One CTA per row, 64-bit radix select on the order-
// preserving image of the double (value desc, lowest column among equals,
// -0 == +0), ascending output.
__global__ void __launch_bounds__(kNT) topk_rows_f64(const double* __restrict__ s, int64_t cols, int64_t keep,
                                                      uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char dsm[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(dsm);
    __shared__ SelSmem sm;
    const int64_t i = blockIdx.x;
    const int n = static_cast<int>(cols);
    for (int j = threadIdx.x; j < n; j += kNT) keys[j] = rank_key_f64(s[i * cols + j]);
    __syncthreads();
    uint64_t T;
    uint32_t rem;
    block_radix_select<uint64_t>(keys, n, static_cast<int>(keep), sm, T, rem);
    block_emit(n, rem, [&](int j, bool& lt, bool& eq) {
        lt = keys[j] < T;
        eq = keys[j] == T;
    }, out + i * keep, sm);
}

// Per-row-scaled top-k (quant_scope = row): the ranking key is
// the double product s_ij * sk_j.  Selection runs on 32-bit keys f =
// fl32(s * sk) (rounding is monotone, so f orders the products except
// inside groups of equal f), then the threshold group is resolved exactly:
// if only part of the f == T group is kept, its members are ranked by the
// double product (ties: lowest column) -- half the radix passes of a 64-bit
// select and the same result.
template <int KD>
__device__ __forceinline__ void topk_row_scaled(const SelectArgs& a, int64_t pair, int64_t i, unsigned char* dsm) {
    const int L = static_cast<int>(a.L);
    uint32_t* keys = reinterpret_cast<uint32_t*>(dsm);            // [L]
    int32_t* ties = reinterpret_cast<int32_t*>(keys + L);          // [L]
    int16_t* sv = reinterpret_cast<int16_t*>(ties + L);            // [L] exact scores
    uint8_t* take = reinterpret_cast<uint8_t*>(sv + L);            // [L]
    __shared__ SelSmem s;
    __shared__ unsigned tie_count;
    const int tid = threadIdx.x;
    const double* skp = a.sk + pair * a.L;
    float q[KD];
    load_levels<KD>(a.lq + pair * a.L * KD, a.L, i, q);
    const uint16_t* lk = a.lk + pair * a.L * KD;
    if (tid == 0) tie_count = 0u;
    for (int j = tid; j < L; j += kNT) {
        const int sc = score_with<KD>(q, lk, a.L, j);
        sv[j] = static_cast<int16_t>(sc);
        take[j] = 0;
        const float f = static_cast<float>(static_cast<double>(sc) * __ldg(skp + j));
        const uint32_t b = __float_as_uint(f == 0.f ? 0.f : f);
        const uint32_t o = (b >> 31) ? ~b : (b | 0x80000000u);  // ascending with f
        keys[j] = ~o;                                           // smaller = better
    }
    __syncthreads();
    uint32_t T, rem;
    block_radix_select<uint32_t>(keys, L, static_cast<int>(a.keep), s, T, rem);
    for (int j = tid; j < L; j += kNT)
        if (keys[j] == T) ties[atomicAdd(&tie_count, 1u)] = j;
    __syncthreads();
    const int m = static_cast<int>(tie_count);
    for (int c = tid; c < m; c += kNT) {
        const int j = ties[c];
        if (static_cast<uint32_t>(m) == rem) {
            take[j] = 1;
            continue;
        }
        const double d = static_cast<double>(sv[j]) * __ldg(skp + j);
        uint32_t rank = 0;
        for (int c2 = 0; c2 < m; ++c2) {
            const int j2 = ties[c2];
            const double d2 = static_cast<double>(sv[j2]) * __ldg(skp + j2);
            rank += (d2 > d || (d2 == d && j2 < j)) ? 1u : 0u;
        }
        take[j] = rank < rem;
    }
    __syncthreads();
    uint32_t* out = a.cols + (pair * a.L + i) * a.keep;
    block_emit(L, 0u, [&](int j, bool& lt, bool& eq) {
        lt = keys[j] < T || (keys[j] == T && take[j]);
        eq = false;
    }, out, s);
}

// rows = blockIdx (grid L x pairs), or the rows listed in `list` (pair * L +
// row, count *nlist; grid-stride) -- the overflow fallback of topk_rowsel.
template <int KD>
__global__ void __launch_bounds__(kNT) topk_rows_scaled(SelectArgs a, const int64_t* list, const unsigned* nlist) {
    extern __shared__ __align__(16) unsigned char dsm[];
    if (list == nullptr) {
        topk_row_scaled<KD>(a, blockIdx.y, blockIdx.x, dsm);
        return;
    }
    const unsigned n = *nlist;
    for (unsigned idx = blockIdx.x; idx < n; idx += gridDim.x) {
        const int64_t g = list[idx];
        topk_row_scaled<KD>(a, g / a.L, g % a.L, dsm);
        __syncthreads();
    }
}

// -------------------------------------------------------------- colvec
template <int KD>
__global__ void __launch_bounds__(kNT) colvec_generic(SelectArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    uint32_t* keys = reinterpret_cast<uint32_t*>(dsm);
    __shared__ SelSmem s;
    const int64_t b = blockIdx.x, pair = blockIdx.y;
    const int L = static_cast<int>(a.L);
    const int64_t r0 = b * a.vec_v, r1 = min(r0 + a.vec_v, a.L);
    const uint16_t* lk = a.lk + pair * a.L * KD;
    const uint16_t* lq = a.lq + pair * a.L * KD;
    for (int j = threadIdx.x; j < L; j += kNT) {
        float kk[KD];
        load_levels<KD>(lk, a.L, j, kk);
        int best = INT32_MIN;
        for (int64_t r = r0; r < r1; ++r) {
            float q[KD];
            load_levels<KD>(lq, a.L, r, q);
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < KD; ++t) acc = fmaf(q[t], kk[t], acc);
            best = max(best, static_cast<int>(acc));
        }
        keys[j] = rank_key_i32(best);
    }
    __syncthreads();
    uint32_t T, rem;
    block_radix_select<uint32_t>(keys, L, static_cast<int>(a.keep), s, T, rem);
    uint32_t* out = a.cols + (pair * ((a.L + a.vec_v - 1) / a.vec_v) + b) * a.keep;
    block_emit(L, rem, [&](int j, bool& lt, bool& eq) {
        lt = keys[j] < T;
        eq = keys[j] == T;
    }, out, s);
}

// --------------------------------------------------------------- block
// pooled[pair][0|1][nb][KD] = sum of the block's rows of levels (exact int).
// Block sums of the levels: one thread per (pair, tensor, block, 8-column
// chunk); the chunk-planar layout makes a block's rows of one chunk a
// contiguous run, read as 16-byte vectors (8 independent sums).
__global__ void pool_levels_kernel(SelectArgs a, int64_t nb) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nch = a.KD / 8;
    const int64_t total = a.pairs * 2 * nb * nch;
    if (idx >= total) return;
    const int64_t c = idx % nch, blk = (idx / nch) % nb, which = (idx / (nch * nb)) % 2,
                  pair = idx / (nch * nb * 2);
    const uint16_t* lv = (which ? a.lk : a.lq) + pair * a.L * a.KD + lvl_index(a.L, 0, static_cast<int>(c * 8));
    int acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int64_t r1 = min((blk + 1) * a.block, a.L);
#pragma unroll 8
    for (int64_t r = blk * a.block; r < r1; ++r) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(lv + r * 8));
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            acc[2 * h] += static_cast<int>(__uint_as_float(ww[h] << 16));
            acc[2 * h + 1] += static_cast<int>(__uint_as_float(ww[h] & 0xffff0000u));
        }
    }
    int32_t* out = a.pooled + ((pair * 2 + which) * nb + blk) * a.KD + c * 8;
#pragma unroll
    for (int u = 0; u < 8; ++u) out[u] = acc[u];
}

__global__ void __launch_bounds__(kNT) block_generic(SelectArgs a, int64_t nb) {
    extern __shared__ __align__(16) unsigned char dsm[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(dsm);
    __shared__ SelSmem s;
    const int64_t ib = blockIdx.x, pair = blockIdx.y;
    const int32_t* pq = a.pooled + ((pair * 2 + 0) * nb + ib) * a.KD;
    const int32_t* pk = a.pooled + (pair * 2 + 1) * nb * a.KD;
    const int64_t r = a.L - (nb - 1) * a.block;  // width of the last (possibly ragged) block
    for (int64_t jb = threadIdx.x; jb < nb; jb += kNT) {
        int64_t sum = 0;
        for (int t = 0; t < a.KD; ++t) sum += static_cast<int64_t>(pq[t]) * pk[jb * a.KD + t];
        const int64_t width = jb == nb - 1 ? r : a.block;
        // mean ranking, exactly: common denominator block * r
        const int64_t val = width == a.block ? sum * r : sum * a.block;
        // 2 val keeps the key odd (INT64_MAX is odd), so the forced diagonal's 0 stays
        // unique without folding neighbouring values together (r = 1: val = sum)
        keys[jb] = (a.force_diag && jb == ib) ? 0ull : rank_key_i64(2 * val);
    }
    __syncthreads();
    uint64_t T;
    uint32_t rem;
    block_radix_select<uint64_t>(keys, static_cast<int>(nb), static_cast<int>(a.keep), s, T, rem);
    uint32_t* out = a.cols + (pair * nb + ib) * a.keep;
    block_emit(static_cast<int>(nb), rem, [&](int j, bool& lt, bool& eq) {
        lt = keys[j] < T;
        eq = keys[j] == T;
    }, out, s);
}

// Warp-per-block-row BLOCK selection (L % block == 0, nb <= 32 * NPL,
// keep <= 32): each lane scores NPL block columns exactly (int32 dot of the
// pooled levels -- with equal block widths the mean ranks like the sum),
// packed as (biased score << 32 | ~block) so one unsigned 64-bit max is
// "value desc, lowest block first"; `keep` rounds of a warp arg-max (the
// forced diagonal ranks above everything) and a 32-lane bitonic sort give
// the ascending block list.  Same ranking as block_generic / the oracle.
// A CTA (8 warps) takes kBRows consecutive block rows of one pair, the
// pair's pooled K staged ONCE in shared memory (row jb's 16-byte chunk t4 at
// position (t4 + jb) mod KD/4, so the 32 lanes' rows spread over the banks).
constexpr int kBRows = 32;
template <int KD, int NPL>
__global__ void __launch_bounds__(256) block_select_warp(SelectArgs a, int64_t nb) {
    extern __shared__ __align__(16) int4 pk_s[];  // [nb][KD / 4], rotated
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t pair = blockIdx.y;
    {
        const int4* pks = reinterpret_cast<const int4*>(a.pooled + (pair * 2 + 1) * nb * KD);
        for (int i = threadIdx.x; i < nb * (KD / 4); i += 256) {
            const int jb = i / (KD / 4), t4 = i % (KD / 4);
            pk_s[jb * (KD / 4) + ((t4 + jb) & (KD / 4 - 1))] = __ldg(pks + i);
        }
    }
    __syncthreads();
    for (int64_t ib = static_cast<int64_t>(blockIdx.x) * kBRows + warp; ib < nb && ib < (blockIdx.x + 1) * static_cast<int64_t>(kBRows); ib += 8) {
    const int32_t* pq = a.pooled + ((pair * 2 + 0) * nb + ib) * KD;
    int32_t qv[KD];
#pragma unroll
    for (int t = 0; t < KD; ++t) qv[t] = __ldg(pq + t);
    unsigned long long key[NPL];
#pragma unroll
    for (int u = 0; u < NPL; ++u) {
        const int jb = u * 32 + lane;
        key[u] = 0ull;
        if (jb < nb) {
            int32_t sum = 0;
            const int4* row = pk_s + jb * (KD / 4);
#pragma unroll
            for (int t4 = 0; t4 < KD / 4; ++t4) {
                const int4 w = row[(t4 + jb) & (KD / 4 - 1)];
                sum += qv[4 * t4] * w.x + qv[4 * t4 + 1] * w.y + qv[4 * t4 + 2] * w.z + qv[4 * t4 + 3] * w.w;
            }
            const uint32_t hi = (a.force_diag && jb == ib) ? 0xffffffffu : (static_cast<uint32_t>(sum) ^ 0x80000000u);
            key[u] = (static_cast<unsigned long long>(hi) << 32) | (0xffffffffu - static_cast<uint32_t>(jb));
        }
    }
    int mine = INT32_MAX;  // lane t keeps the t-th selected block
    for (int k = 0; k < static_cast<int>(a.keep); ++k) {
        unsigned long long best = key[0];
#pragma unroll
        for (int u = 1; u < NPL; ++u) best = key[u] > best ? key[u] : best;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, off);
            best = o > best ? o : best;
        }
        if (lane == k) mine = static_cast<int>(0xffffffffu - static_cast<uint32_t>(best));
#pragma unroll
        for (int u = 0; u < NPL; ++u)
            if (key[u] == best) key[u] = 0ull;  // unique: only the owner's slot matches
    }
    // ascending order: bitonic sort across the 32 lanes
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const int other = __shfl_xor_sync(0xffffffffu, mine, stride);
            const bool up = (lane & size) == 0;
            const bool lower = (lane & stride) == 0;
            mine = (lower == up) ? min(mine, other) : max(mine, other);
        }
    }
    if (lane < a.keep) a.cols[(pair * nb + ib) * a.keep + lane] = static_cast<uint32_t>(mine);
    }
}

// ----------------------------------------------------------- threshold
// E[pair][t] = rint(det_exp(c * -t) * 2^40), c = s_q s_k / sqrt(d).
__global__ void exp_table_kernel(SelectArgs a) {
    const int64_t pair = blockIdx.y;
    const double c = a.sq[pair] * a.sk[pair] / sqrt(static_cast<double>(a.D));
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < a.span;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double e = det_exp(c * static_cast<double>(-t));
        a.etab[pair * a.span + t] = static_cast<int64_t>(rint(e * 1099511627776.0));
    }
}

__device__ __forceinline__ bool keep_rule(uint64_t e, uint64_t z, uint64_t ln, uint64_t den) {
    // e * ln >= z * den, exact in 128 bits
    const uint64_t lh = __umul64hi(e, ln), ll = e * ln;
    const uint64_t rh = __umul64hi(z, den), rl = z * den;
    return lh != rh ? lh > rh : ll >= rl;
}

// emit == 0: write the kept count to counts[pair*L + i]; emit == 1: write
// the kept columns at rowptr[pair*L + i].
template <int KD>
__global__ void __launch_bounds__(kNT) threshold_generic(SelectArgs a, uint64_t* counts, int emit) {
    extern __shared__ __align__(16) unsigned char dsm[];
    uint32_t* keys = reinterpret_cast<uint32_t*>(dsm);
    __shared__ SelSmem s;
    const int64_t i = blockIdx.x, pair = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = a.causal ? static_cast<int>(i) + 1 : static_cast<int>(a.L);
    float q[KD];
    load_levels<KD>(a.lq + pair * a.L * KD, a.L, i, q);
    const uint16_t* lk = a.lk + pair * a.L * KD;
    int mx = INT32_MIN;
    for (int j = tid; j < n; j += kNT) {
        const int sc = score_with<KD>(q, lk, a.L, j);
        keys[j] = static_cast<uint32_t>(sc);
        mx = max(mx, sc);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if (lane == 0) s.red[warp] = static_cast<unsigned long long>(static_cast<uint32_t>(mx));
    __syncthreads();
    int M = INT32_MIN;
    for (int w = 0; w < kWarps; ++w) M = max(M, static_cast<int>(static_cast<uint32_t>(s.red[w])));
    __syncthreads();
    const int64_t* E = a.etab + pair * a.span;
    unsigned long long z = 0;
    for (int j = tid; j < n; j += kNT) z += static_cast<unsigned long long>(__ldg(E + (M - static_cast<int>(keys[j]))));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
    if (lane == 0) s.red[warp] = z;
    __syncthreads();
    unsigned long long Z = 0;
    for (int w = 0; w < kWarps; ++w) Z += s.red[w];
    __syncthreads();
    const uint64_t ln = static_cast<uint64_t>(a.L) * static_cast<uint64_t>(a.frac_num);
    const uint64_t den = static_cast<uint64_t>(a.frac_den);
    // rank keys: kept -> rank_key_i32(score) (< UINT32_MAX), dropped -> UINT32_MAX
    unsigned cnt_local = 0;
    for (int j = tid; j < n; j += kNT) {
        const int sc = static_cast<int>(keys[j]);
        const bool kept = keep_rule(static_cast<uint64_t>(__ldg(E + (M - sc))), Z, ln, den);
        keys[j] = kept ? rank_key_i32(sc) : 0xffffffffu;
        cnt_local += kept;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) cnt_local += __shfl_xor_sync(0xffffffffu, cnt_local, off);
    if (lane == 0) s.red[warp] = cnt_local;
    __syncthreads();
    uint32_t cnt = 0;
    for (int w = 0; w < kWarps; ++w) cnt += static_cast<uint32_t>(s.red[w]);
    __syncthreads();
    const uint32_t take = cnt > static_cast<uint32_t>(a.cap) ? static_cast<uint32_t>(a.cap) : cnt;
    if (!emit) {
        if (tid == 0) {
            counts[pair * a.L + i] = take;
            if (a.empty_rows) a.empty_rows[pair * a.L + i] = take == 0;
        }
        return;
    }
    uint32_t* out = a.cols + a.rowptr[pair * a.L + i];
    if (cnt <= static_cast<uint32_t>(a.cap)) {
        block_emit(n, 0u, [&](int j, bool& lt, bool& eq) {
            lt = keys[j] != 0xffffffffu;
            eq = false;
        }, out, s);
    } else {
        uint32_t T, rem;
        block_radix_select<uint32_t>(keys, n, static_cast<int>(a.cap), s, T, rem);
        block_emit(n, rem, [&](int j, bool& lt, bool& eq) {
            lt = keys[j] < T;
            eq = keys[j] == T;
        }, out, s);
    }
}

template <int KD>
void launch_select(const SelectArgs& a, cudaStream_t st) {
    const unsigned P = static_cast<unsigned>(a.pairs);
    switch (a.mode) {
        case kRowTopk: {
            if (a.per_row && a.L <= 8192 && a.qmax * a.qmax * KD < 32768) {  // int16 exact scores
                const size_t sm = static_cast<size_t>(a.L) * 11;
                auto kern = topk_rows_scaled<KD>;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
                kern<<<dim3(static_cast<unsigned>(a.L), P), kNT, sm, st>>>(a, nullptr, nullptr);
                note_launch();
            } else if (a.per_row) {
                const size_t sm = static_cast<size_t>(a.L) * 8;
                auto kern = topk_rows_generic<uint64_t, KD>;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
                kern<<<dim3(static_cast<unsigned>(a.L), P), kNT, sm, st>>>(a);
                note_launch();
            } else {
                const size_t sm = static_cast<size_t>(a.L) * 4;
                auto kern = topk_rows_generic<uint32_t, KD>;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
                kern<<<dim3(static_cast<unsigned>(a.L), P), kNT, sm, st>>>(a);
                note_launch();
            }
            break;
        }
        case kColvec: {
            const size_t sm = static_cast<size_t>(a.L) * 4;
            auto kern = colvec_generic<KD>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
            kern<<<dim3(static_cast<unsigned>(ceil_div_i(a.L, a.vec_v)), P), kNT, sm, st>>>(a);
                note_launch();
            break;
        }
        case kBlock: {
            const int64_t nb = ceil_div_i(a.L, a.block);
            const int64_t total = a.pairs * 2 * nb * (a.KD / 8);
            pool_levels_kernel<<<static_cast<unsigned>(ceil_div_i(total, 256)), 256, 0, st>>>(a, nb);
            note_launch();
            const double bq = static_cast<double>(a.block) * a.qmax;  // |pooled level| bound
            const bool warp_ok = a.keep <= 32 && a.L % a.block == 0 && nb <= 512 &&
                                 static_cast<double>(a.KD) * bq * bq < 2147483647.0 &&  // int32 dot exact
                                 !options().block_generic;
            const dim3 gw(static_cast<unsigned>(ceil_div_i(nb, kBRows)), P);
            const size_t psm = static_cast<size_t>(nb) * KD * 4;  // pooled K of the pair
            auto bsw = [&](auto kern) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(psm));
                kern<<<gw, 256, psm, st>>>(a, nb);
            };
            if (warp_ok && nb <= 128) {
                bsw(block_select_warp<KD, 4>);
            } else if (warp_ok && nb <= 256) {
                bsw(block_select_warp<KD, 8>);
            } else if (warp_ok) {
                bsw(block_select_warp<KD, 16>);
            } else {
                const size_t sm = static_cast<size_t>(nb) * 8;
                cudaFuncSetAttribute(block_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
                block_generic<<<dim3(static_cast<unsigned>(nb), P), kNT, sm, st>>>(a, nb);
            }
            note_launch();
            break;
        }
        case kThreshold: {
            launch_exp_table(a, st);
            const size_t sm = static_cast<size_t>(a.L) * 4;
            auto kern = threshold_generic<KD>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
            kern<<<dim3(static_cast<unsigned>(a.L), P), kNT, sm, st>>>(a, a.counts, 0);
            note_launch();
            scan_counts(a, st);
            kern<<<dim3(static_cast<unsigned>(a.L), P), kNT, sm, st>>>(a, a.counts, 1);
            note_launch();
            break;
        }
        default: throw_unsupported("unknown mask mode");
    }
}

}  // namespace

void launch_exp_table(const SelectArgs& a, cudaStream_t st) {
    exp_table_kernel<<<dim3(static_cast<unsigned>(std::min<int64_t>(ceil_div_i(a.span, 256), 64)),
                            static_cast<unsigned>(a.pairs)), 256, 0, st>>>(a);
    note_launch();
}

// rowptr[0] = 0, rowptr[1..] = inclusive scan of the per-row kept counts
void scan_counts(const SelectArgs& a, cudaStream_t st) {
    cudaMemsetAsync(a.rowptr, 0, sizeof(uint64_t), st);
    size_t tb = a.scan_tmp_bytes;
    cub::DeviceScan::InclusiveSum(a.scan_tmp, tb, a.counts, a.rowptr + 1, static_cast<int64_t>(a.pairs * a.L), st);
}

void run_row_topk_f64(const double* s, int64_t rows, int64_t cols, int64_t keep, uint32_t* out, cudaStream_t st) {
    if (rows == 0) return;
    const size_t sm = static_cast<size_t>(cols) * 8;
    cudaFuncSetAttribute(topk_rows_f64, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    topk_rows_f64<<<static_cast<unsigned>(rows), kNT, sm, st>>>(s, cols, keep, out);
    note_launch();
}

void launch_topk_scaled_list(const SelectArgs& a, const int64_t* list, const unsigned* nlist, cudaStream_t st) {
    const size_t sm = static_cast<size_t>(a.L) * 11;
    const unsigned grid = 148 * 4;  // grid-stride over the (normally empty) list
    if (a.KD == 16) {
        cudaFuncSetAttribute(topk_rows_scaled<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
        topk_rows_scaled<16><<<grid, kNT, sm, st>>>(a, list, nlist);
    } else {
        cudaFuncSetAttribute(topk_rows_scaled<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
        topk_rows_scaled<32><<<grid, kNT, sm, st>>>(a, list, nlist);
    }
    note_launch();
}

size_t select_scan_tmp_bytes(int64_t n) {
    size_t b = 0;
    cub::DeviceScan::InclusiveSum(nullptr, b, static_cast<const uint64_t*>(nullptr),
                                  static_cast<uint64_t*>(nullptr), n);
    return b;
}

void run_select(const SelectArgs& a, cudaStream_t st) {
    if (colvec_tc_supported(a)) {
        run_colvec_tc(a, st);
        return;
    }
    if (threshold_tc_supported(a)) {
        run_threshold_tc(a, st);
        return;
    }
    if (topk_rowsel_supported(a)) {
        run_topk_rowsel(a, st);
        return;
    }
    switch (a.KD) {
        case 16: launch_select<16>(a, st); break;
        case 32: launch_select<32>(a, st); break;
        default: throw_unsupported("projection width k must be 16 or 32");
    }
}

}  // namespace dsa
