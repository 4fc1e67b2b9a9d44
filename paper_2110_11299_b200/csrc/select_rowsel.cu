// Phase 2 fast path for per-row top-k with per-row scales (ROW_TOPK,
// quant_scope = row; C1): one warp per query row, the row's keys
// held in registers, a single windowed histogram instead of a radix select.
//
// Reference: predicted_topk_mask -> row_topk_indices (P/src/maskgen.cpp:18-20,
// P/src/linalg.cpp:69-85): keep the `keep` largest rank keys of a row, ties
// to the LOWEST column, output ascending.  With per-row scales the rank key
// is the double product d_j = S_int[i][j] * s_k[j] (oracle
// dsa_oracle_mask_topk_rowscaled; s_q[i] is a positive row constant).
//
// A CTA stages one pair's K~ levels as int8 rows in shared memory (exact:
// |level| <= 127) and each warp walks its rows.  Lane l owns the NPL
// CONSECUTIVE keys j = l*NPL + u (rows XOR-swizzled so the 16-byte loads of
// a warp are conflict-free), so its kept keys come out in ascending order
// and one warp scan places every lane's run.  Per row:
//
//   1  scores: s = <q~, k~_j> (DP4A), f_j = fl32(s) * fl32(s_k[j]) -- within
//      2^-23 |d_j| of the exact key; row max M; the maximum of each group of
//      NPL/G keys (32*G >= keep groups)
//   2  f_lo = min over the 32*G group maxima: count(f >= f_lo) >= keep, so the
//      keep-th largest lies in [f_lo, M].  Bins of width w = (M - f_lo)/250
//      below M: t_j = round((M - f_j)/w) (one FFMA, magic-number rounding),
//      a warp-private 256-bin histogram of the t_j < 256 (shared atomics,
//      keys below the window skipped)
//   3  b = the bin holding the keep-th key.  Since w >> the fl32 error,
//      t_j <= b-2  -> certainly kept (fewer than keep keys can outrank it)
//      t_j >= b+2  -> certainly dropped (>= keep keys rank strictly above)
//      t_j in b-1..b+1 -> candidates, ranked by the EXACT double key (ties:
//      lowest column); the best keep - #kept of them are taken
//   4  emission: per-lane counts -> warp exclusive scan -> each lane writes
//      its kept columns in order.
//
// Rows whose window is degenerate (w not >> the fl32 error) or whose
// candidate set exceeds kCand go to the overflow list, finished by the
// CTA-per-row kernel (normally none).
#include <cuda_bf16.h>

#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"

namespace dsa {
namespace {

constexpr int kWarps = 8;
constexpr int kChunk = 256;  // query rows staged per chunk
constexpr int kBins = 256;
constexpr int kCand = 256;
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: float -> integer by rounding
constexpr int kMagicBits = 0x4B400000;

struct RowSelWarp {
    uint32_t hist[kBins];
    uint32_t chosen[64];  // candidate keys taken (bit per column, L <= 2048)
    double dval[kCand];
    uint16_t cand[kCand];
    uint32_t ncand;
    uint32_t pad[3];
};

__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// 8 bf16 levels (one 16-byte chunk) -> 8 packed int8
__device__ __forceinline__ uint2 pack_levels(uint4 w) {
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
    uint32_t b[2] = {0u, 0u};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const int lo = static_cast<int>(__uint_as_float(ww[h] << 16));
        const int hi = static_cast<int>(__uint_as_float(ww[h] & 0xffff0000u));
        b[h >> 1] |= ((static_cast<uint32_t>(lo) & 0xffu) | ((static_cast<uint32_t>(hi) & 0xffu) << 8)) << ((h & 1) * 16);
    }
    return make_uint2(b[0], b[1]);
}

template <int KD>
__device__ __forceinline__ int dot_i8(const int (&q)[KD / 4], const int4* kr) {
    int s = 0;
#pragma unroll
    for (int v = 0; v < KD / 16; ++v) {
        const int4 w = kr[v];
        s = __dp4a(q[4 * v], w.x, s);
        s = __dp4a(q[4 * v + 1], w.y, s);
        s = __dp4a(q[4 * v + 2], w.z, s);
        s = __dp4a(q[4 * v + 3], w.w, s);
    }
    return s;
}

// row j of the staged K~ lives in slot j ^ ((j / NPL) & 7)
template <int NPL>
__device__ __forceinline__ int slot_of(int j) {
    return j ^ ((j / NPL) & 7);
}

template <int KD, int NPL, int G>
__global__ void __launch_bounds__(kWarps * 32, 2) topk_rowsel_kernel(SelectArgs a) {
    static_assert(NPL % 8 == 0 && NPL % G == 0 && NPL <= 64, "layout");
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr int L = 32 * NPL;
    constexpr int kGS = NPL / G;  // keys per group
    int8_t* kl = reinterpret_cast<int8_t*>(dsm);                       // [L][KD] swizzled rows
    float* skt = reinterpret_cast<float*>(dsm + L * KD);                // [NPL][32]
    RowSelWarp* wsm = reinterpret_cast<RowSelWarp*>(dsm + L * KD + L * 4);
    int8_t* qs = reinterpret_cast<int8_t*>(dsm + L * KD + L * 4 + kWarps * sizeof(RowSelWarp));  // [kChunk][KD]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    RowSelWarp& ws = wsm[warp];
    const uint32_t keep = static_cast<uint32_t>(a.keep);
    const int xl = lane & 7;
    const int4* krow[8];  // lane's rows u = 8v + e live at slot base + 8v + (e ^ xl)
#pragma unroll
    for (int e = 0; e < 8; ++e)
        krow[e] = reinterpret_cast<const int4*>(kl + (lane * NPL + (e ^ xl)) * KD);
    const float* skl = skt + lane;

    // persistent: CTA b owns the flattened (pair, row) range [r0, r1), walked
    // in chunks of <= kChunk rows of one pair; K~ is restaged on pair change
    const int64_t total = a.pairs * L;
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * per;
    const int64_t r1 = r0 + per < total ? r0 + per : total;
    int64_t staged = -1;
    for (int64_t c0 = r0; c0 < r1;) {
        const int64_t pair = c0 / L;
        const int row0 = static_cast<int>(c0 - pair * L);
        int n = L - row0;
        if (n > kChunk) n = kChunk;
        if (n > r1 - c0) n = static_cast<int>(r1 - c0);
        const uint16_t* lqp = a.lq + pair * L * KD;
        const double* skp = a.sk + pair * L;
        __syncthreads();  // the previous chunk is done with the staged rows
        if (pair != staged) {
            // K~ as int8 (consecutive threads: consecutive rows of one chunk)
            const uint16_t* lkp = a.lk + pair * L * KD;
            for (int t = tid; t < L * (KD / 8); t += kWarps * 32) {
                const int r = t % L, c = t / L;
                const uint4 w = __ldg(reinterpret_cast<const uint4*>(lkp + lvl_index(L, r, c * 8)));
                *reinterpret_cast<uint2*>(kl + slot_of<NPL>(r) * KD + c * 8) = pack_levels(w);
            }
            for (int j = tid; j < L; j += kWarps * 32) skt[(j % NPL) * 32 + j / NPL] = static_cast<float>(__ldg(skp + j));
            staged = pair;
        }
        for (int t = tid; t < n * (KD / 8); t += kWarps * 32) {
            const int r = t % n, c = t / n;
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(lqp + lvl_index(L, row0 + r, c * 8)));
            *reinterpret_cast<uint2*>(qs + r * KD + c * 8) = pack_levels(w);
        }
        __syncthreads();
        c0 += n;
        for (int rr = warp; rr < n; rr += kWarps) {
            const int i = row0 + rr;
            int q[KD / 4];
#pragma unroll
            for (int v = 0; v < KD / 16; ++v) {
                const int4 w = reinterpret_cast<const int4*>(qs + rr * KD)[v];
                q[4 * v] = w.x;
                q[4 * v + 1] = w.y;
                q[4 * v + 2] = w.z;
                q[4 * v + 3] = w.w;
            }
            // ---- 1: scores, lane max, group maxima
            float f[NPL];
            float gm[G];
#pragma unroll
            for (int u = 0; u < NPL; ++u) {
                const int s = dot_i8<KD>(q, krow[u & 7] + (u & ~7) * (KD / 16));
                f[u] = static_cast<float>(s) * skl[u * 32];
                if (u % kGS == 0) gm[u / kGS] = f[u];
                else gm[u / kGS] = fmaxf(gm[u / kGS], f[u]);
            }
            float lmax = gm[0], lmin = gm[0];
#pragma unroll
            for (int g = 1; g < G; ++g) {
                lmax = fmaxf(lmax, gm[g]);
                lmin = fminf(lmin, gm[g]);
            }
            const float M = warp_max(lmax);
            const float flo = warp_min(lmin);
            // ---- 2: window histogram
            const float w = (M - flo) * (1.0f / 250.0f);
            const float mag = fmaxf(fabsf(M), fabsf(flo));
            bool ovf = !(w >= mag * 6.103515625e-05f) || !(w > 0.f);  // w >= 2^-14 |key|
            uint32_t b = 0, nA = 0;
            if (!ovf) {
                const float ninv = -1.0f / w;
                // +2: every key lands in a bin >= 1 whatever the rounding of c0
                const float c0 = fmaf(M, -ninv, kMagic) + 2.0f;
                {
                    uint4* h4 = reinterpret_cast<uint4*>(ws.hist);
                    h4[lane * 2] = make_uint4(0u, 0u, 0u, 0u);
                    h4[lane * 2 + 1] = make_uint4(0u, 0u, 0u, 0u);
                    ws.chosen[lane] = 0u;
                    ws.chosen[lane + 32] = 0u;
                }
                __syncwarp();
                // the key is replaced by its biased bin bits kMagicBits + t (t >= 1)
                const uint32_t hbase = static_cast<uint32_t>(__cvta_generic_to_shared(ws.hist)) -
                                       static_cast<uint32_t>(kMagicBits) * 4u;
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const int tb = __float_as_int(__fmaf_rn(f[u], ninv, c0));
                    f[u] = __int_as_float(tb);
                    if (tb < kMagicBits + kBins)
                        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hbase + static_cast<uint32_t>(tb) * 4u) : "memory");
                }
                __syncwarp();
                // ---- 3: bin of the keep-th key
                const uint4 h0 = reinterpret_cast<const uint4*>(ws.hist)[lane * 2];
                const uint4 h1 = reinterpret_cast<const uint4*>(ws.hist)[lane * 2 + 1];
                const uint32_t hb[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
                uint32_t tot = 0;
#pragma unroll
                for (int e = 0; e < 8; ++e) tot += hb[e];
                uint32_t incl = tot;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += y;
                }
                const uint32_t excl = incl - tot;
                const bool mine = excl < keep && keep <= incl;
                const unsigned who = __ballot_sync(0xffffffffu, mine);
                uint32_t bsel = 0;
                if (mine) {
                    uint32_t cum = excl;
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        if (bsel == 0u && cum + hb[e] >= keep) bsel = static_cast<uint32_t>(lane * 8 + e) + 1u;
                        cum += hb[e];
                    }
                }
                ovf = who == 0u;
                b = __shfl_sync(0xffffffffu, bsel, who ? __ffs(who) - 1 : 0) - 1u;
                if (!ovf) {
                    // counts of bins <= b-2 (kept) and b-1..b+1 (candidates)
                    uint32_t ca = 0, cc = 0;
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int bin = lane * 8 + e;
                        ca += bin + 2 <= static_cast<int>(b) ? hb[e] : 0u;
                        cc += (bin + 1 >= static_cast<int>(b) && bin <= static_cast<int>(b) + 1) ? hb[e] : 0u;
                    }
                    nA = __reduce_add_sync(0xffffffffu, ca);
                    const uint32_t nc = __reduce_add_sync(0xffffffffu, cc);
                    ovf = nc > static_cast<uint32_t>(kCand);
                }
            }
            uint32_t* out = a.cols + (pair * L + i) * a.keep;
            if (!ovf) {
                // ---- collect candidates, count certain keys per lane
                const int bC = kMagicBits + static_cast<int>(b) - 1;
                uint32_t ma[(NPL + 31) / 32] = {};  // certainly kept keys (bit u)
                uint32_t mc[(NPL + 31) / 32] = {};  // candidates (bit u)
#pragma unroll
                for (int u = 0; u < NPL; ++u) {
                    const int d = __float_as_int(f[u]) - bC;
                    if (d < 0) ma[u >> 5] |= 1u << (u & 31);
                    if (static_cast<unsigned>(d) < 3u) mc[u >> 5] |= 1u << (u & 31);
                }
                {
                    uint32_t nl = 0;
#pragma unroll
                    for (int x = 0; x < (NPL + 31) / 32; ++x) nl += static_cast<uint32_t>(__popc(mc[x]));
                    uint32_t inc = nl;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, off);
                        if (lane >= off) inc += y;
                    }
                    uint32_t slot = inc - nl;
                    if (lane == 31) ws.ncand = inc;
#pragma unroll
                    for (int x = 0; x < (NPL + 31) / 32; ++x) {
                        uint32_t m = mc[x];
                        while (m) {
                            const int u = __ffs(m) - 1;
                            m &= m - 1u;
                            ws.cand[slot++] = static_cast<uint16_t>(lane * NPL + x * 32 + u);
                        }
                    }
                }
                __syncwarp();
                const uint32_t nc = ws.ncand;
                const uint32_t need = keep - nA;
                // exact keys of the candidates
                for (uint32_t c = lane; c < nc; c += 32) {
                    const int j = ws.cand[c];
                    const int s = dot_i8<KD>(q, reinterpret_cast<const int4*>(kl + slot_of<NPL>(j) * KD));
                    ws.dval[c] = static_cast<double>(s) * __ldg(skp + j);
                }
                __syncwarp();
                for (uint32_t c = lane; c < nc; c += 32) {
                    const int j = ws.cand[c];
                    const double d = ws.dval[c];
                    uint32_t rank = 0;
                    for (uint32_t c2 = 0; c2 < nc; ++c2) {
                        const double d2 = ws.dval[c2];
                        const int j2 = ws.cand[c2];
                        rank += (d2 > d || (d2 == d && j2 < j)) ? 1u : 0u;
                    }
                    if (rank < need) atomicOr(&ws.chosen[j >> 5], 1u << (j & 31));
                }
                __syncwarp();
                uint32_t cm[(NPL + 31) / 32];
                if (NPL >= 32) {
#pragma unroll
                    for (int x = 0; x < NPL / 32; ++x) cm[x] = ws.chosen[lane * (NPL / 32) + x] | ma[x];
                } else {
                    cm[0] = ((ws.chosen[(lane * NPL) >> 5] >> ((lane * NPL) & 31)) & ((1u << (NPL & 31)) - 1u)) | ma[0];
                }
                uint32_t n_l = 0;
#pragma unroll
                for (int x = 0; x < (NPL + 31) / 32; ++x) n_l += static_cast<uint32_t>(__popc(cm[x]));
                uint32_t incl = n_l;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += y;
                }
                // ---- 4: emission in ascending column order
                uint32_t* o = out + (incl - n_l);
#pragma unroll
                for (int x = 0; x < (NPL + 31) / 32; ++x) {
                    uint32_t m = cm[x];
                    while (m) {
                        const int u = __ffs(m) - 1;
                        m &= m - 1u;
                        *o++ = static_cast<uint32_t>(lane * NPL + x * 32 + u);
                    }
                }
            } else if (lane == 0) {
                const unsigned slot = atomicAdd(a.ovf_n, 1u);
                a.ovf_list[slot] = pair * L + i;
            }
            __syncwarp();
        }
    }
}

template <int KD, int NPL, int G>
void launch_rowsel(const SelectArgs& a, cudaStream_t st) {
    constexpr int L = 32 * NPL;
    const size_t smem = static_cast<size_t>(L) * (KD + 4) + kWarps * sizeof(RowSelWarp) + kChunk * KD;
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t total = a.pairs * L;
    const int64_t grid = std::min<int64_t>(2 * sms, ceil_div_i(total, 64));
    auto kern = topk_rowsel_kernel<KD, NPL, G>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<static_cast<unsigned>(grid), kWarps * 32, smem, st>>>(a);
    note_launch();
}

template <int KD, int NPL>
void dispatch_g(const SelectArgs& a, cudaStream_t st) {
    if (a.keep <= 32) launch_rowsel<KD, NPL, 1>(a, st);
    else if (a.keep <= 64) launch_rowsel<KD, NPL, 2>(a, st);
    else if (a.keep <= 128) launch_rowsel<KD, NPL, 4>(a, st);
    else launch_rowsel<KD, NPL, 8>(a, st);
}

template <int KD>
void dispatch_rowsel(const SelectArgs& a, cudaStream_t st) {
    switch (a.L) {
        case 512: dispatch_g<KD, 16>(a, st); break;
        case 1024: dispatch_g<KD, 32>(a, st); break;
        default: dispatch_g<KD, 64>(a, st); break;
    }
}

}  // namespace

bool topk_rowsel_supported(const SelectArgs& a) {
    if (a.mode != kRowTopk || !a.per_row || a.ovf_n == nullptr) return false;
    if (a.KD != 16 && a.KD != 32) return false;
    if (a.L != 512 && a.L != 1024 && a.L != 2048) return false;  // L = 32 * NPL
    const int64_t npl = a.L / 32;
    // 32 * G groups >= keep with G <= 8 and G | NPL
    if (a.keep < 1 || a.keep > 256 || a.keep > 32 * std::min<int64_t>(8, npl)) return false;
    if (a.qmax > 127) return false;  // int8 levels
    return !options().topk_generic;
}

void run_topk_rowsel(const SelectArgs& a, cudaStream_t st) {
    cudaMemsetAsync(a.ovf_n, 0, sizeof(unsigned), st);
    if (a.KD == 16) dispatch_rowsel<16>(a, st);
    else dispatch_rowsel<32>(a, st);
    launch_topk_scaled_list(a, a.ovf_list, a.ovf_n, st);  // overflow rows (normally none)
}

}  // namespace dsa
