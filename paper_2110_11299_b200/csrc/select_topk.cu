// Phase 2 fast path for per-row top-k with per-row scales (ROW_TOPK,
// quant_scope = row; C1): tcgen05 scores + a per-thread exact
// selection on the double rank key d_j = s_ij * sk_j (oracle
// dsa_oracle_mask_topk_rowscaled; ties to the lowest column).
//
// One CTA owns 128 query rows (thread = row = TMEM lane, rowscore_tc.cuh).
// The approximate key fa = s * fl32(sk_j) is within 2 ulps of the exact
// product, so its order-preserving integer o(fa) orders the keys except
// within a few ulps.  Passes over the key tiles:
//   1  O_max / O_min of o(fa)
//   2  64-bin histogram of D = O_max - o over the row's range  -> bin b1
//      holding the keep-th largest
//   3  64 sub-bins of b1                                     -> sub-bin b2
//   4  collect C = { D <= edge(b2) + 8 ulps } (ascending columns, exact
//      scores) into a per-thread list: every exact top-keep key is in C
//      (anything outside has >= keep keys more than 8 ulps above it)
// then the |C| - keep worst members of C by the exact double key (ties:
// highest column first) are dropped and the row is written.  Rows whose C
// exceeds the list (pathological ties) go to an overflow list finished by
// the CTA-per-row kernel.  Opt-in (DSA_TOPK_TC=1): on C1 the refinement
// levels (8 bits each over a ~2^31-wide ordered range) cost up to six passes
// of ~15 instructions per score, slower than the CTA-per-row radix select.
#include <cuda_bf16.h>

#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"
#include "rowscore_tc.cuh"
#include "tc_sm100.cuh"

namespace dsa {
namespace {

using namespace rs;

constexpr int kBins = 256;  // per level (8 bits of the ordered key), u16 counters packed in pairs
constexpr int kExtra = 64;  // list slots beyond keep

struct TopkParams {
    const uint16_t* lq;
    const uint16_t* lk;
    const double* sk;  // [pairs][L]
    int64_t L, keep;
    uint32_t* cols;    // [pairs][L][keep]
    unsigned* ovf_n;
    int64_t* ovf_list;  // pair * L + row
};

__device__ __forceinline__ uint32_t ord32(float f) {
    const uint32_t b = __float_as_uint(f == 0.f ? 0.f : f);
    return (b >> 31) ? ~b : (b | 0x80000000u);
}

template <int KD>
struct TopkLayout {
    static constexpr int kQ = kTQ * KD * 2;
    static constexpr int kTile = kTN * KD * 2;
    __host__ __device__ static int region(int64_t keep) {  // histogram / candidate list (disjoint lifetimes)
        const int hist = (kBins / 2) * kTQ * 4;
        const int list = static_cast<int>(keep + kExtra) * kTQ * 4;
        return hist > list ? hist : list;
    }
    static int bytes(int64_t L, int64_t keep) {
        return kQ + kSt * kTile + static_cast<int>((L + 3) & ~int64_t{3}) * 4 + region(keep) + 64;
    }
};

template <int KD>
__global__ void __launch_bounds__(kTQ) topk_tc_kernel(TopkParams a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    using Ly = TopkLayout<KD>;
    const int64_t L = a.L;
    const int keep = static_cast<int>(a.keep);
    const int cap = keep + kExtra;
    unsigned char* bq = smem;
    unsigned char* ring = bq + Ly::kQ;
    float* skf = reinterpret_cast<float*>(ring + kSt * Ly::kTile);
    unsigned char* region = reinterpret_cast<unsigned char*>(skf + ((L + 3) & ~int64_t{3}));  // 16-B aligned
    uint32_t* hist = reinterpret_cast<uint32_t*>(region);  // [bin][thread]
    uint32_t* clist = reinterpret_cast<uint32_t*>(region);  // [slot][thread]: col << 16 | (uint16) s
    uint64_t* bars = reinterpret_cast<uint64_t*>(region + Ly::region(a.keep));
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t pair = blockIdx.y;
    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * kTQ;
    const int64_t row = q0 + tid;
    const bool rvalid = row < L;
    const double* skp = a.sk + pair * L;

    if (tid == 0) {
        tc::mbar_init(&bars[0], 1);
        tc::mbar_init(&bars[1], 1);
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<2 * kTN>(tslot);
    for (int64_t j = tid; j < L; j += kTQ) skf[j] = static_cast<float>(__ldg(skp + j));
    load_rows<KD, kTQ>(tc::smem_addr(bq), a.lq + pair * L * KD, q0, L, tid);
    cp_commit();
    cp_wait<0>();
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
    c.nkt = static_cast<int>((L + kTN - 1) / kTN);
    c.tid = tid;
    c.warp = warp;
    uint32_t g = 0;

    // ---- pass 1: range of o(fa)
    uint32_t omax = 0u, omin = 0xffffffffu;
    score_pass<KD>(c, g, [&](int u, const uint32_t* r, int col0) {
        const float* f = reinterpret_cast<const float*>(r);
        const int64_t k0 = static_cast<int64_t>(u) * kTN + col0;
        const int lim = k0 + 32 <= L ? 32 : static_cast<int>(L - k0);
#pragma unroll
        for (int x = 0; x < 32; ++x) {
            const uint32_t o = ord32(f[x] * skf[k0 + x < L ? k0 + x : 0]);
            if (x < lim) {
                omax = max(omax, o);
                omin = min(omin, o);
            }
        }
    });
    const uint32_t range = omax - omin;
    const int s1 = range < kBins ? 0 : (32 - __clz(range) - 8);  // (range >> s1) < 256
    uint32_t* hcol = hist + tid;
    // ---- passes 2..: 64 bins of D = omax - o over [lo, lo + 64 << sh), then
    // 64 sub-bins of the bin holding the keep-th largest, until that bin
    // holds few keys (or single ulps)
    uint32_t lo = 0u, before = 0u, edge = 0u;
    int sh = s1;
    bool active = true;
    auto bin_count = [&](int b) -> uint32_t { return (hcol[(b >> 1) * kTQ] >> ((b & 1) << 4)) & 0xffffu; };
    while (__syncthreads_or(active)) {
        for (int i = tid; i < (kBins / 2) * kTQ; i += kTQ) hist[i] = 0u;
        __syncthreads();
        score_pass<KD>(c, g, [&](int u, const uint32_t* r, int col0) {
            if (!active) return;
            const float* f = reinterpret_cast<const float*>(r);
            const int64_t k0 = static_cast<int64_t>(u) * kTN + col0;
            const int lim = k0 + 32 <= L ? 32 : static_cast<int>(L - k0);
#pragma unroll
            for (int x = 0; x < 32; ++x) {
                const uint32_t D = omax - ord32(f[x] * skf[k0 + x < L ? k0 + x : 0]);
                const uint32_t bin = (D - lo) >> sh;
                if (x < lim && D >= lo && bin < kBins) atomicAdd(hcol + (bin >> 1) * kTQ, 1u << ((bin & 1) << 4));
            }
        });
        if (active) {
            int b = 0;
            uint32_t h = 0;
            for (; b < kBins; ++b) {
                h = bin_count(b);
                if (before + h >= static_cast<uint32_t>(keep)) break;
                before += h;
            }
            if (b >= kBins) {  // cannot happen (keep <= L); be safe: take everything
                b = kBins - 1;
                h = 0xffffu;
            }
            edge = lo + ((static_cast<uint32_t>(b) + 1u) << sh) - 1u;
            if (sh == 0 || h <= 16u) {
                active = false;
            } else {
                lo += static_cast<uint32_t>(b) << sh;
                sh = sh > 8 ? sh - 8 : 0;
            }
        }
        __syncthreads();
    }
    __syncthreads();  // histogram region becomes the candidate lists
    // ---- pass 4: candidates D <= edge + 8 (saturating), ascending columns
    const uint32_t lim_d = edge > 0xffffffffu - 8u ? 0xffffffffu : edge + 8u;
    int n = 0;
    bool ovf = false;
    uint32_t* mylist = clist + tid;
    score_pass<KD>(c, g, [&](int u, const uint32_t* r, int col0) {
        const float* f = reinterpret_cast<const float*>(r);
        const int64_t k0 = static_cast<int64_t>(u) * kTN + col0;
        const int lim = k0 + 32 <= L ? 32 : static_cast<int>(L - k0);
#pragma unroll
        for (int x = 0; x < 32; ++x) {
            const uint32_t d = omax - ord32(f[x] * skf[k0 + x < L ? k0 + x : 0]);
            if (x < lim && d <= lim_d) {
                // column << 16 | exact integer score (|s| < 2^15)
                if (n < cap) mylist[n * kTQ] = (static_cast<uint32_t>(k0 + x) << 16) |
                                               (static_cast<uint32_t>(static_cast<int>(f[x])) & 0xffffu);
                else ovf = true;
                ++n;
            }
        }
    });
    __syncthreads();
    if (rvalid && ovf) {
        const unsigned slot = atomicAdd(a.ovf_n, 1u);
        a.ovf_list[slot] = pair * L + row;
    }
    if (rvalid && !ovf) {
        auto key_of = [&](uint32_t e) -> double {
            const int j = static_cast<int>(e >> 16);
            const int sc = static_cast<int>(static_cast<int16_t>(e & 0xffffu));
            return static_cast<double>(sc) * __ldg(skp + j);
        };
        // drop the n - keep worst (smallest key; among equal keys the highest column)
        for (int dpos = n; dpos > keep; --dpos) {
            int worst = -1;
            double wk = 0.0;
            uint32_t wj = 0;
            for (int t = 0; t < n; ++t) {
                const uint32_t e = mylist[t * kTQ];
                if (e == 0xffffffffu) continue;
                const double k = key_of(e);
                const uint32_t j = e >> 16;
                if (worst < 0 || k < wk || (k == wk && j > wj)) {
                    worst = t;
                    wk = k;
                    wj = j;
                }
            }
            mylist[worst * kTQ] = 0xffffffffu;
        }
        uint32_t* out = a.cols + (pair * L + row) * a.keep;
        int o = 0;
        for (int t = 0; t < n; ++t) {
            const uint32_t e = mylist[t * kTQ];
            if (e != 0xffffffffu) out[o++] = e >> 16;
        }
    }
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<2 * kTN>(c.tmem);
}

}  // namespace

bool topk_tc_supported(const SelectArgs& a) {
    if (a.mode != kRowTopk || !a.per_row || a.ovf_n == nullptr) return false;
    if (a.KD != 16 && a.KD != 32) return false;
    if (a.L > 65535 || a.keep > 160) return false;       // 16-bit columns in the lists
    if (a.qmax * a.qmax * a.KD >= 32768) return false;    // 16-bit exact scores
    // opt-in: correct (parity-tested) but measured slower than the CTA-per-row
    // radix kernel on C1 (4.5 vs 2.9 ms): up to six passes over the scores
    if (std::getenv("DSA_TOPK_TC") == nullptr) return false;
    const int bytes = a.KD == 16 ? TopkLayout<16>::bytes(a.L, a.keep) : TopkLayout<32>::bytes(a.L, a.keep);
    return bytes <= 200 * 1024;
}

void run_topk_tc(const SelectArgs& a, cudaStream_t st) {
    TopkParams p{};
    p.lq = a.lq;
    p.lk = a.lk;
    p.sk = a.sk;
    p.L = a.L;
    p.keep = a.keep;
    p.cols = a.cols;
    p.ovf_n = a.ovf_n;
    p.ovf_list = a.ovf_list;
    cudaMemsetAsync(a.ovf_n, 0, sizeof(unsigned), st);
    const dim3 grid(static_cast<unsigned>(ceil_div_i(a.L, kTQ)), static_cast<unsigned>(a.pairs));
    if (a.KD == 16) {
        const int smem = TopkLayout<16>::bytes(a.L, a.keep);
        cudaFuncSetAttribute(topk_tc_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        topk_tc_kernel<16><<<grid, kTQ, smem, st>>>(p);
    } else {
        const int smem = TopkLayout<32>::bytes(a.L, a.keep);
        cudaFuncSetAttribute(topk_tc_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        topk_tc_kernel<32><<<grid, kTQ, smem, st>>>(p);
    }
    note_launch();
    launch_topk_scaled_list(a, a.ovf_list, a.ovf_n, st);  // overflow rows (normally none)
}

}  // namespace dsa
