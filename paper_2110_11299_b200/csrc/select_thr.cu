// Phase 2 fast path for threshold masks (SURVEY 8(a) O4 / maskgen.cpp:22-31):
// tcgen05 score GEMM fused with the exact integer threshold rule.
//
// One CTA owns 128 query rows of one (b,h) pair; the 5th-gen tensor core
// produces the exact integer scores
//
//   D[q, key] = sum_c Q~[q, c] * K~[key, c]     tcgen05.mma kind::f16, M = 128
//                                               queries, N = 64 keys, K = 16
//
// into TMEM (double-buffered, 2 x 64 columns; three count / four emit CTAs
// per SM).  Every
// thread owns one TMEM lane = one query row, so all per-row reductions are
// in-thread.  The rule (keep j iff E[m - s_j] * L * num >= Z * den, with
// E[t] = rint(exp(-c t) 2^40), Z = sum_j E[m - s_j], then the `cap` highest
// scores, ties to the lowest index; oracle dsa_oracle_mask_threshold) needs
// the row max before anything else, so the key tiles are streamed in passes:
//
//   count kernel:  pass 1  row max m                          (FMNMX3)
//                  pass 2  per-thread histogram of t = m - s over the first
//                          kW bins (Z from it; keys beyond the bins with
//                          E[t] > 0 only bound Z, and a rare extra pass sums
//                          them exactly when the bound leaves t* ambiguous)
//                  -> t* (largest kept t, binary search on E), kept count,
//                     cap cut and tie quota from the histogram prefix sums;
//                     rows whose cut lies beyond kW bins run extra counting
//                     passes (binary search on the cut) -- exact, rare
//   scan           rowptr = exclusive scan of the kept counts (cub)
//   emit kernel:   pass 3  keys with s > v_cut, then the first `quota` keys
//                          with s == v_cut, in ascending key order (each
//                          thread writes its own row's list)
//
// The L x L score matrix never exists in HBM; K~ tiles are the only
// streamed operand (bulk cp.async into a 3-stage ring).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>
#include <type_traits>

#include "device_common.cuh"
#include "kernels.h"
#include "rowscore_tc.cuh"
#include "tc_sm100.cuh"

namespace dsa {
namespace {

using namespace rs;

constexpr int kW = 119;   // histogram bins per row (t = m - s in [0, kW)); 30 KB -> 4 CTAs/SM
constexpr int kHC = kTQ / 2;  // histogram columns: rows r and r + 64 share a word (16-bit halves)
constexpr uint32_t kAll = 0xffffffffu;
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: float -> int by addition
constexpr int kMagicBits = 0x4B400000;

__device__ __forceinline__ bool keep_rule(uint64_t e, uint64_t z, uint64_t ln, uint64_t den) {
    const uint64_t lh = __umul64hi(e, ln), ll = e * ln;
    const uint64_t rh = __umul64hi(z, den), rl = z * den;
    return lh != rh ? lh > rh : ll >= rl;
}

struct ThrParams {
    const uint16_t* lq;
    const uint16_t* lk;
    const int64_t* etab;  // [pairs][span]
    int64_t span, L, cap;
    int causal;
    int faddr;            // KD * qmax^2 < 15000: one-FFMA bin addresses (pass 2)
    uint64_t ln, den;     // L * frac_num, frac_den
    uint64_t* counts;     // [pairs * L]
    int2* cut;            // [pairs * L]: {v_cut, quota}
    uint8_t* empty_rows;
    const uint64_t* rowptr;
    uint32_t* cols;
};

template <int KD>
struct ThrLayout {
    static constexpr int kQ = kTQ * KD * 2;
    static constexpr int kTile = kTN * KD * 2;
    static constexpr int kHist = (kW + 1) * kHC * 4;  // [bin][row % 64] + trash bin: each warp conflict-free
    static constexpr int kE = kW * 8;
    static constexpr int bytes(bool emit) { return kQ + kSt * kTile + (emit ? 0 : kHist + kE) + 64; }
};

// P16 (emit only, KD * qmax^2 <= 2048): scores in an f16 accumulator, two
// keys per packed compare (see rs::score_pass)
template <int KD, bool EMIT, bool P16 = false>
__global__ void __launch_bounds__(kTQ, 4) threshold_tc_kernel(ThrParams a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    using Ly = ThrLayout<KD>;
    unsigned char* bq = smem;
    unsigned char* ring = bq + Ly::kQ;
    unsigned char* p = ring + kSt * Ly::kTile;
    uint32_t* hist = reinterpret_cast<uint32_t*>(p);
    uint64_t* es = reinterpret_cast<uint64_t*>(p + (EMIT ? 0 : Ly::kHist));
    uint64_t* bars = reinterpret_cast<uint64_t*>(p + (EMIT ? 0 : Ly::kHist + Ly::kE));
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
    int* tz_s = reinterpret_cast<int*>(bars + 3);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t L = a.L;
    const int nqt = static_cast<int>((L + kTQ - 1) / kTQ);
    const int64_t q0 = static_cast<int64_t>(nqt - 1 - static_cast<int>(blockIdx.x)) * kTQ;  // heavy tiles first
    const int64_t pair = blockIdx.y;
    const int64_t row = q0 + tid;
    const bool rvalid = row < L;
    const int64_t kend = a.causal ? (q0 + kTQ < L ? q0 + kTQ : L) : L;
    // keys up to this bound are valid for every row of the CTA
    const int64_t kfree = a.causal ? q0 + 1 : L;

    if (tid == 0) {
        tc::mbar_init(&bars[0], 1);
        tc::mbar_init(&bars[1], 1);
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<2 * kTN>(tslot);
    const int64_t* E = a.etab + pair * a.span;
    if (!EMIT) {
        for (int t = tid; t < kW; t += kTQ) es[t] = t < a.span ? static_cast<uint64_t>(__ldg(E + t)) : 0ull;
        for (int t = tid; t < (kW + 1) * kHC; t += kTQ) hist[t] = 0u;
        if (tid == 0) {  // tz = first t with E[t] == 0 (E is non-increasing), or span
            int64_t lo = 0, hi = a.span;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (__ldg(E + mid) == 0) hi = mid;
                else lo = mid + 1;
            }
            *tz_s = static_cast<int>(lo);
        }
    }
    load_rows<KD, kTQ>(tc::smem_addr(bq), a.lq + pair * L * KD, q0, L, tid);
    cp_commit();
    cp_wait<0>();
    if (P16) cvt_rows_f16<KD, kTQ>(bq, tid);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();

    PassCtx c;
    c.ring = ring;
    c.bars = bars;
    c.tmem = *tslot;
    c.qdesc = tc::desc_kmajor_nosw(tc::smem_addr(bq), 128, KD * 16);
    c.lkp = a.lk + pair * L * KD;
    c.L = L;
    c.nkt = static_cast<int>((kend + kTN - 1) / kTN);
    c.tid = tid;
    c.warp = warp;
    uint32_t g = 0;
    const int64_t gi = pair * L + row;

    // valid(key) for this thread's row: key < kend and (causal: key <= row)
    const int64_t klim = a.causal ? row + 1 : L;  // keys < klim are candidates

    if (!EMIT) {
        // ---- pass 1: row max
        float m = -INFINITY;
        score_pass<KD>(c, g, [&](int u, const uint32_t* r, int col0) {
            const float* f = reinterpret_cast<const float*>(r);
            const int64_t k0 = static_cast<int64_t>(u) * kTN + col0;
            if (k0 + 32 <= kfree) {
#pragma unroll
                for (int x = 0; x < 32; x += 2) {
                    float y;
                    asm("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(m), "f"(f[x]), "f"(f[x + 1]));
                    m = y;
                }
            } else {
#pragma unroll
                for (int x = 0; x < 32; ++x)
                    if (k0 + x < klim) m = fmaxf(m, f[x]);
            }
        });
        // ---- pass 2: histogram of t = m - s over bins [0, wh), wh = min(tz, kW);
        // every other key (t >= wh, and masked keys) lands in the trash bin wh
        const int tz = *tz_s;
        const int wh = tz < kW ? tz : kW;
        const float mb = m + kMagic;
        // row tid counts in the low (tid < 64) or high 16-bit half of word
        // [bin][tid % 64] (a row has < 65536 candidate keys)
        uint32_t* hcol = hist + (tid & (kHC - 1));
        const uint32_t hinc = tid < kHC ? 1u : 0x10000u;
        const int hsh = tid < kHC ? 0 : 16;
        {
            // The bin ADDRESS comes out of one FFMA in the subnormal range:
            // with D(n) = n * 2^-149 (bit pattern n), D(-256) * s + D(A)
            // with A = col address + 256 m is exactly D(A - 256 s) = D(col
            // address + 256 t) -- every term is an integer multiple of
            // 2^-149 below 2^-126, so the product and the sum are exact
            // (fma.rn without .ftz keeps subnormals).  Bits of positive
            // floats are monotone, so an unsigned min clamps to the trash
            // bin (t >= wh, the masked keys' -inf -> +inf).  FFMA + VIMNMX
            // + ATOMS per key instead of FADD + VIMNMX + IMAD + ATOMS.
            const uint32_t cbase = tc::smem_addr(hcol);
            const uint32_t lim = cbase + static_cast<uint32_t>(wh) * (kHC * 4u);
            const float dneg = __uint_as_float(0x80000000u | (kHC * 4u));  // -D(256)
            // A = cbase + 256 m as a signed subnormal (|A| < 2^23 when faddr)
            const int32_t A = static_cast<int32_t>(cbase) + __float2int_rn(m) * static_cast<int32_t>(kHC * 4);
            const float dA = __uint_as_float(A >= 0 ? static_cast<uint32_t>(A) : (0x80000000u | static_cast<uint32_t>(-A)));
            // otherwise: bin bits = kMagicBits + t (float magic) and one IMAD
            const uint32_t mlim = static_cast<uint32_t>(kMagicBits + wh);
            const uint32_t abase = cbase - static_cast<uint32_t>(kMagicBits) * (kHC * 4u);
            // two instantiations of the pass (no per-key branch)
            auto hist_pass = [&](auto FA) {
            score_pass<KD>(c, g, [&](int u, const uint32_t* r, int col0) {
                const float* f = reinterpret_cast<const float*>(r);
                const int64_t k0 = static_cast<int64_t>(u) * kTN + col0;
                auto one = [&](float v) {
                    uint32_t addr;
                    if (decltype(FA)::value) {
                        float d;
                        asm("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(v), "f"(dneg), "f"(dA));
                        addr = min(__float_as_uint(d), lim);
                    } else {
                        addr = min(__float_as_uint(fmaf(v, -1.0f, mb)), mlim) * (kHC * 4u) + abase;
                    }
                    // shared-memory reduction without return value: no
                    // load -> add -> store chain between consecutive keys
                    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(hinc) : "memory");
                };
                if (k0 + 32 <= kfree) {
#pragma unroll
                    for (int x = 0; x < 32; ++x) one(f[x]);
                } else {
#pragma unroll
                    for (int x = 0; x < 32; ++x) one(k0 + x < klim ? f[x] : -INFINITY);
                }
            });
            };
            if (a.faddr) hist_pass(std::true_type{});
            else hist_pass(std::false_type{});
        }
        // ---- per-row rule from the histogram
        auto bin = [&](int t) -> uint32_t { return (hcol[t * kHC] >> hsh) & 0xffffu; };
        uint64_t Z = 0;
        uint32_t htot = 0;
        for (int t = 0; t < wh; ++t) {
            const uint32_t h = bin(t);
            Z += static_cast<uint64_t>(h) * es[t];
            htot += h;
        }
        // t* = largest t with E[t] kept (E non-increasing); -1: nothing kept
        auto tstar_of = [&](uint64_t Zv) -> int {
            if (!rvalid || !keep_rule(es[0], Zv, a.ln, a.den)) return -1;
            int lo = 0, hi = tz - 1;  // keep_rule(E[lo]) holds; E[tz] == 0 never kept
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                const uint64_t e = mid < kW ? es[mid] : static_cast<uint64_t>(__ldg(E + mid));
                if (keep_rule(e, Zv, a.ln, a.den)) lo = mid;
                else hi = mid - 1;
            }
            return lo;
        };
        // keys beyond the bins with E[t] > 0 (t in [kW, tz), tz > kW) add at
        // most E[kW] each: Z lies in [Z, Z + trash * E[kW]].  When both ends
        // give the same t*, it is exact; otherwise (rare) one more pass sums
        // those E[t] exactly.
        int tstar = tstar_of(Z);
        bool amb = false;
        if (tz > wh && rvalid) {
            const uint64_t zhi = Z + static_cast<uint64_t>(bin(wh)) * static_cast<uint64_t>(__ldg(E + wh));
            amb = tstar_of(zhi) != tstar;
        }
        if (__syncthreads_or(amb)) {
            uint64_t zt = 0;
            const uint32_t span = static_cast<uint32_t>(tz - wh);
            score_pass<KD>(c, g, [&](int u, const uint32_t* r, int col0) {
                if (!amb) return;
                const float* f = reinterpret_cast<const float*>(r);
                const int64_t k0 = static_cast<int64_t>(u) * kTN + col0;
                for (int y = 0; y < 32; ++y) {
                    const int t = __float_as_int(fmaf(f[y], -1.0f, mb)) - kMagicBits;
                    if (k0 + y < klim && static_cast<uint32_t>(t - wh) < span)
                        zt += static_cast<uint64_t>(__ldg(E + t));
                }
            });
            if (amb) {
                Z += zt;
                tstar = tstar_of(Z);
            }
        }
        const uint32_t cap = static_cast<uint32_t>(a.cap);
        uint32_t take = 0, quota = kAll;
        int cut = -1;  // keep t < cut, plus `quota` of t == cut (kAll: all of them)
        int st = 0;    // 1: count(t <= t*) needed, 2: binary search for the cap cut
        int x = 0, lo = 0, hi = 0;
        uint32_t clo = 0;
        if (tstar >= 0) {
            if (tstar < kW || htot >= cap) {
                const int lim = tstar < kW ? tstar : kW - 1;
                uint32_t pre = 0;
                int t = 0;
                for (; t <= lim; ++t) {
                    const uint32_t h = bin(t);
                    if (pre + h >= cap) break;
                    pre += h;
                }
                if (t > lim) {  // count(t <= t*) = pre <= cap... (tstar < kW here)
                    take = pre;
                    cut = tstar;
                } else if (pre + bin(t) == cap && t == tstar) {
                    take = cap;
                    cut = tstar;
                } else {
                    take = cap;
                    cut = t;
                    quota = cap - pre;
                }
            } else {
                st = 1;
                x = tstar;
            }
        }
        // rare: the cut lies beyond the histogram -> counting passes
        while (__syncthreads_or(st != 0)) {
            uint32_t cnt = 0;
            score_pass<KD>(c, g, [&](int u, const uint32_t* r, int col0) {
                if (!st) return;
                const float* f = reinterpret_cast<const float*>(r);
                const int64_t k0 = static_cast<int64_t>(u) * kTN + col0;
#pragma unroll
                for (int y = 0; y < 32; ++y) {
                    const int t = __float_as_int(fmaf(f[y], -1.0f, mb)) - kMagicBits;
                    cnt += (t <= x && k0 + y < klim) ? 1u : 0u;
                }
            });
            if (st == 1) {
                if (cnt <= cap) {
                    take = cnt;
                    cut = tstar;
                    st = 0;
                } else {
                    st = 2;
                    lo = kW - 1;
                    clo = htot;
                    hi = tstar;
                }
            } else if (st == 2) {
                if (cnt >= cap) hi = x;
                else {
                    lo = x;
                    clo = cnt;
                }
            }
            if (st == 2) {
                if (hi == lo + 1) {
                    take = cap;
                    cut = hi;
                    quota = cap - clo;
                    st = 0;
                } else {
                    x = (lo + hi) >> 1;
                }
            }
        }
        if (rvalid) {
            a.counts[gi] = take;
            // v_cut = m - cut as a score; nothing kept -> above every score
            const int mi = __float2int_rn(m);
            a.cut[gi] = make_int2(take == 0 ? INT32_MAX : mi - cut, static_cast<int>(quota));
            if (a.empty_rows) a.empty_rows[gi] = take == 0;
        }
    } else {
        // ---- emission: s > v_cut, then the first `quota` with s == v_cut
        int2 ci = make_int2(INT32_MAX, 0);
        uint32_t* out = a.cols;
        if (rvalid) {
            ci = a.cut[gi];
            out += a.rowptr[gi];
        }
        const float vc = ci.x == INT32_MAX ? INFINITY : static_cast<float>(ci.x);
        uint32_t quota = static_cast<uint32_t>(ci.y);
        uint32_t n = 0;
        // keep the first `quota` set bits of eq (ties, lowest key first)
        auto ties = [&](uint32_t ge, uint32_t eq) -> uint32_t {
            eq &= ge;
            uint32_t keq = eq;
            const uint32_t ne = static_cast<uint32_t>(__popc(eq));
            if (ne > quota) {
                keq = 0;
                uint32_t e = eq;
                for (uint32_t i = 0; i < quota; ++i) {
                    keq |= e & (~e + 1u);
                    e &= e - 1u;
                }
            }
            quota -= static_cast<uint32_t>(__popc(keq));
            return (ge & ~eq) | keq;
        };
        if (P16) {
            // every score is an integer in [-2048, 2048]: clamping v_cut to
            // that range keeps the comparisons exact in f16
            const float vcl = fminf(fmaxf(vc, -2048.f), 4096.f);
            const __half2 v2 = __half2half2(__float2half_rn(vc > 2048.f ? INFINITY : vcl));
            score_pass<KD, true>(c, g, [&](int u, const uint32_t* r, int) {
                const int64_t kt = static_cast<int64_t>(u) * kTN;
#pragma unroll
                for (int grp = 0; grp < 2; ++grp) {
                    const int64_t k0 = kt + grp * 32;
                    const int lim = k0 + 32 <= kfree ? 32 : static_cast<int>(klim - k0);
                    uint32_t ge = 0;
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const __half2 x = *reinterpret_cast<const __half2*>(&r[grp * 16 + i]);
                        ge |= __hge2_mask(x, v2) & (0x00010001u << i);
                    }
                    if (lim < 32) ge &= lim > 0 ? (0xffffffffu >> (32 - lim)) : 0u;
                    if (quota != kAll && ge) {
                        uint32_t eq = 0;
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const __half2 x = *reinterpret_cast<const __half2*>(&r[grp * 16 + i]);
                            eq |= __heq2_mask(x, v2) & (0x00010001u << i);
                        }
                        ge = ties(ge, eq);
                    }
                    while (ge) {
                        const int y = __ffs(ge) - 1;
                        ge &= ge - 1u;
                        out[n++] = static_cast<uint32_t>(k0 + y);
                    }
                }
            });
        } else
        score_pass<KD>(c, g, [&](int u, const uint32_t* r, int col0) {
            const float* f = reinterpret_cast<const float*>(r);
            const int64_t k0 = static_cast<int64_t>(u) * kTN + col0;
            const int lim = k0 + 32 <= kfree ? 32 : static_cast<int>(klim - k0);
            uint32_t ge = 0;
#pragma unroll
            for (int y = 0; y < 32; ++y) ge |= f[y] >= vc ? (1u << y) : 0u;
            if (lim < 32) ge &= lim > 0 ? (0xffffffffu >> (32 - lim)) : 0u;
            if (quota != kAll && ge) {  // capped row: only the first `quota` ties
                uint32_t eq = 0;
#pragma unroll
                for (int y = 0; y < 32; ++y) eq |= f[y] == vc ? (1u << y) : 0u;
                ge = ties(ge, eq);
            }
            while (ge) {
                const int y = __ffs(ge) - 1;
                ge &= ge - 1u;
                out[n++] = static_cast<uint32_t>(k0 + y);
            }
        });
    }
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<2 * kTN>(c.tmem);
}

template <int KD, bool EMIT, bool P16 = false>
void launch_thr(const ThrParams& p, int64_t pairs, cudaStream_t st) {
    // at least 46 KB so no fifth CTA lands on an SM whose TMEM is taken
    // (TMEM: 4 x 128 columns)
    const int smem = std::max(ThrLayout<KD>::bytes(EMIT), 46 * 1024);
    auto kern = threshold_tc_kernel<KD, EMIT, P16>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const dim3 grid(static_cast<unsigned>(ceil_div_i(p.L, kTQ)), static_cast<unsigned>(pairs));
    kern<<<grid, kTQ, smem, st>>>(p);
    note_launch();
}

}  // namespace

bool threshold_tc_supported(const SelectArgs& a) {
    return a.mode == kThreshold && !a.per_row && (a.KD == 16 || a.KD == 32) && a.L < 65536 - kTN &&  // 16-bit histogram halves
          
           a.cut != nullptr && !options().threshold_generic;
}

// exp table -> count kernel -> scan -> emit kernel
void run_threshold_tc(const SelectArgs& a, cudaStream_t st) {
    ThrParams p{};
    p.lq = a.lq;
    p.lk = a.lk;
    p.etab = a.etab;
    p.span = a.span;
    p.L = a.L;
    p.cap = a.cap;
    p.causal = a.causal;
    p.faddr = a.KD * static_cast<int64_t>(a.qmax) * a.qmax < 15000;
    p.ln = static_cast<uint64_t>(a.L) * static_cast<uint64_t>(a.frac_num);
    p.den = static_cast<uint64_t>(a.frac_den);
    p.counts = a.counts;
    p.cut = a.cut;
    p.empty_rows = a.empty_rows;
    p.rowptr = a.rowptr;
    p.cols = a.cols;
    launch_exp_table(a, st);
    if (a.KD == 16) launch_thr<16, false>(p, a.pairs, st);
    else launch_thr<32, false>(p, a.pairs, st);
    scan_counts(a, st);
    // f16 scores are exact when |S| and every partial sum stay <= 2048
    const bool p16 = a.KD * static_cast<int64_t>(a.qmax) * a.qmax <= 2048;
    if (a.KD == 16) {
        if (p16) launch_thr<16, true, true>(p, a.pairs, st);
        else launch_thr<16, true>(p, a.pairs, st);
    } else {
        if (p16) launch_thr<32, true, true>(p, a.pairs, st);
        else launch_thr<32, true>(p, a.pairs, st);
    }
}

}  // namespace dsa
