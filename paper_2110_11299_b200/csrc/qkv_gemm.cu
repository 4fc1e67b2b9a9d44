// The step before the hot path: the per-head Q/K/V
// projections of one attention layer plus the predictor input, as ONE bf16
// tcgen05 GEMM over X.
//
// Reference: project_qkv (P/src/attention.cpp:36-46) computes, per head h,
// Q_h = X W_Q[h], K_h = X W_K[h], V_h = X W_V[h] with three matmuls that
// each re-read X; the trainer reads X a fourth time for the predictor input
// R = X P (P/src/trainer.cpp:162).  Here the packed weights
// W = [W_Q[0..H) | W_K[0..H) | W_V[0..H) | P]^T  ([n_out][d_model], K-major)
// turn all of it into  Y = X W^T  (M = batch * L rows, N = n_out, K = d_model)
// with the head split fused into the epilogue: Y's columns are scattered
// straight into the [batch*H][L][d] bf16 layout the predict / select /
// attention kernels read (R stays f32: [batch][L][npred]).
//
// Kernel: persistent, warp-specialised, one CTA per SM.
//   warp 0   TMA producer: 128x64 X tiles and 256x64 W tiles (128-byte
//            swizzle) into a 4-stage shared-memory ring (full/empty mbarriers)
//   warp 1   MMA issuer (one thread): tcgen05.mma kind::f16, M = 128,
//            N = 256 (narrower on the last column tile), K = 16 x 4 per
//            stage, fp32 accumulators in TMEM, double-buffered (2 x 256
//            columns) so the epilogue of tile t overlaps the MMAs of t + 1
//   warps 2-5  epilogue: tcgen05.ld 32 columns at a time (thread = output
//            row = TMEM lane), bf16 pack, 64-byte row segments stored to
//            their head's slab.
// Tiles are walked M-major (consecutive CTAs share an X row block, W stays
// L2 resident).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "device_common.cuh"
#include "kernels.h"
#include "tc_sm100.cuh"
#include "tma_map.h"

namespace dsa {
namespace {

constexpr int kBM = 128;   // rows per tile (UMMA M)
constexpr int kBN = 256;   // output columns per tile (UMMA N)
constexpr int kBK = 64;    // K per stage: one 128-byte swizzle atom row
constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK * 2;   // 16 KB
constexpr int kBBytes = kBN * kBK * 2;   // 32 KB
constexpr int kThreads = 192;            // 6 warps
constexpr int kStg = 32 * 128;           // one warp's 32 rows x 64 bf16 staging tile (TMA store)
constexpr int kSmem = kStages * (kABytes + kBBytes) + 4 * 2 * kStg + 1024 + 256;

struct QkvArgs {
    int64_t M, L, H, dk, dv, npred, n_out, kdim;
    __nv_bfloat16* q;
    __nv_bfloat16* k;
    __nv_bfloat16* v;
    float* r;
    int tma_store;  // Q/K/V tiles leave through TMA (d_k, d_v % 64 == 0, L % 32 == 0)
};

// K-major operand tile written by TMA with 128-byte swizzle: rows of 128 B,
// 8-row atoms 1024 B apart (SBO); layout type 2 = SWIZZLE_128B (sm_100
// descriptor bits 61-63), version 1 (bit 46).  K steps of 16 elements advance
// the start address by 32 B inside the atom.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;                 // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;         // SBO
    d |= static_cast<uint64_t>(1) << 46;                 // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2) << 61;                 // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ uint32_t bc_pack(uint32_t lo, uint32_t hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y), "r"(src)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    qkv_gemm_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                    const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, QkvArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the swizzled tiles
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t{1023});
    unsigned char* sa = smem;                                  // [kStages][kABytes]
    unsigned char* sb = smem + kStages * kABytes;              // [kStages][kBBytes]
    unsigned char* stg = sb + kStages * kBBytes;               // [4 warps][2][kStg], 1024-aligned
    uint64_t* bars = reinterpret_cast<uint64_t*>(stg + 4 * 2 * kStg);
    uint64_t* full = bars;               // [kStages] TMA -> MMA
    uint64_t* empty = bars + kStages;    // [kStages] MMA -> TMA
    uint64_t* tfull = bars + 2 * kStages;      // [2] MMA -> epilogue
    uint64_t* tempty = bars + 2 * kStages + 2; // [2] epilogue -> MMA (4 warp arrivals)
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t mt = (a.M + kBM - 1) / kBM;
    const int64_t ntl = (a.n_out + kBN - 1) / kBN;
    const int64_t ntiles = mt * ntl;
    const int nk = static_cast<int>(a.kdim / kBK);

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&tfull[s], 1);
            tc::mbar_init(&tempty[s], 4);
        }
        tc::fence_barrier_init();
    }
    if (warp == 2) tc::tmem_alloc<512>(tslot);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int m0 = static_cast<int>((t / ntl) * kBM);
                const int n0 = static_cast<int>((t % ntl) * kBN);
                for (int kb = 0; kb < nk; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1u);
                    const uint32_t fb = tc::smem_addr(&full[stage]);
                    expect_tx(fb, kABytes + kBBytes);
                    tma_load_2d(tc::smem_addr(sa + stage * kABytes), &map_x, kb * kBK, m0, fb);
                    tma_load_2d(tc::smem_addr(sb + stage * kBBytes), &map_w, kb * kBK, n0, fb);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int64_t n0 = (t % ntl) * kBN;
                int nn = static_cast<int>(std::min<int64_t>(kBN, a.n_out - n0));
                nn = (nn + 15) & ~15;  // UMMA N: multiple of 16 for M = 128
                const uint32_t idesc = tc::idesc_bf16_f32(kBM, nn);
                tc::mbar_wait(&tempty[acc], aphase ^ 1u);  // epilogue drained this accumulator
                tc::fence_after_sync();
                const uint32_t dt = tmem + static_cast<uint32_t>(acc * kBN);
                for (int kb = 0; kb < nk; ++kb) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::fence_after_sync();
                    const uint64_t ad = desc_sw128(tc::smem_addr(sa + stage * kABytes));
                    const uint64_t bd = desc_sw128(tc::smem_addr(sb + stage * kBBytes));
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk)
                        tc::mma_bf16(dt, ad + static_cast<uint64_t>(kk * 2), bd + static_cast<uint64_t>(kk * 2), idesc,
                                     (kb | kk) != 0);
                    tc::commit(&empty[stage]);  // frees the smem slot when these MMAs finish
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                tc::commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    aphase ^= 1u;
                }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2-5)
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int64_t HK = a.H * a.dk, HV = a.H * a.dv;
        int acc = 0, sbuf = 0;
        uint32_t aphase = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int64_t m0 = (t / ntl) * kBM;
            const int64_t n0 = (t % ntl) * kBN;
            const int ncols = static_cast<int>(std::min<int64_t>(kBN, a.n_out - n0));
            tc::mbar_wait(&tfull[acc], aphase);
            tc::fence_after_sync();
            const int64_t m = m0 + quarter * 32 + lane;
            const bool mvalid = m < a.M;
            const int64_t b = mvalid ? m / a.L : 0, l = mvalid ? m - b * a.L : 0;
            const uint32_t tbase = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * kBN);
            int c0 = 0;
            // TMA-store path: this warp's 32 rows lie in one batch row block,
            // so each 64-column head chunk is a [32][64] box of the head's slab
            const int64_t mw = m0 + quarter * 32;
            if (a.tma_store && mw + 32 <= a.M && (mw % a.L) + 32 <= a.L) {
                const int64_t bw = mw / a.L, lw = mw - bw * a.L;
                for (; c0 < ncols && n0 + c0 < 2 * HK + HV; c0 += 64) {
                    uint32_t r0[32], r1[32];
                    tc::ld_32x32b_x32(tbase + c0, r0);
                    tc::ld_32x32b_x32(tbase + c0 + 32, r1);
                    tc::wait_ld();
                    const int64_t n = n0 + c0;
                    const CUtensorMap* map;
                    int64_t y;
                    int x;
                    if (n < HK) {
                        map = &map_q;
                        y = (bw * a.H + n / a.dk) * a.L + lw;
                        x = static_cast<int>(n % a.dk);
                    } else if (n < 2 * HK) {
                        map = &map_k;
                        y = (bw * a.H + (n - HK) / a.dk) * a.L + lw;
                        x = static_cast<int>((n - HK) % a.dk);
                    } else {
                        map = &map_v;
                        y = (bw * a.H + (n - 2 * HK) / a.dv) * a.L + lw;
                        x = static_cast<int>((n - 2 * HK) % a.dv);
                    }
                    // the staging buffer's previous TMA store has read its bytes
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
                    __syncwarp();
                    unsigned char* st = stg + ((warp - 2) * 2 + sbuf) * kStg;
                    const uint32_t sro = tc::smem_addr(st) + lane * 128;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {  // 128-byte swizzle: chunk j of row r at j ^ (r & 7)
                        const uint32_t* rr = j < 4 ? &r0[8 * j] : &r1[8 * (j - 4)];
                        const uint32_t w0 = bc_pack(rr[0], rr[1]), w1 = bc_pack(rr[2], rr[3]);
                        const uint32_t w2 = bc_pack(rr[4], rr[5]), w3 = bc_pack(rr[6], rr[7]);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(sro + ((j ^ (lane & 7)) << 4)),
                                     "r"(w0), "r"(w1), "r"(w2), "r"(w3)
                                     : "memory");
                    }
                    tc::fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) tma_store_2d(map, x, static_cast<int>(y), tc::smem_addr(st));
                    sbuf ^= 1;
                }
            }
            for (; c0 < ncols; c0 += 32) {
                uint32_t r[32];
                tc::ld_32x32b_x32(tbase + c0, r);
                tc::wait_ld();
                if (!mvalid) continue;
                const int64_t n = n0 + c0;  // 32-column chunk inside one head / region
                if (n < 2 * HK + HV) {
                    __nv_bfloat16* dst;
                    if (n < HK) {
                        dst = a.q + ((b * a.H + n / a.dk) * a.L + l) * a.dk + n % a.dk;
                    } else if (n < 2 * HK) {
                        const int64_t nn2 = n - HK;
                        dst = a.k + ((b * a.H + nn2 / a.dk) * a.L + l) * a.dk + nn2 % a.dk;
                    } else {
                        const int64_t nn2 = n - 2 * HK;
                        dst = a.v + ((b * a.H + nn2 / a.dv) * a.L + l) * a.dv + nn2 % a.dv;
                    }
                    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        uint4 w;
                        w.x = bc_pack(r[8 * s + 0], r[8 * s + 1]);
                        w.y = bc_pack(r[8 * s + 2], r[8 * s + 3]);
                        w.z = bc_pack(r[8 * s + 4], r[8 * s + 5]);
                        w.w = bc_pack(r[8 * s + 6], r[8 * s + 7]);
                        d4[s] = w;
                    }
                } else if (a.r) {
                    const int64_t pc = n - 2 * HK - HV;
                    float* dst = a.r + m * a.npred + pc;
                    for (int x = 0; x < 32 && pc + x < a.npred; ++x) dst[x] = __uint_as_float(r[x]);
                }
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) arrive(tc::smem_addr(&tempty[acc]));
            if (++acc == 2) {
                acc = 0;
                aphase ^= 1u;
            }
        }
    }
    if (warp >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    __syncthreads();
    if (warp == 2) tc::tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ host
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeFn>(p);
    }();
    return fn;
}

}  // namespace

// 2-D bf16 row-major [rows][cols] -> box [box_rows][box_cols] with 128-byte swizzle
CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int box_rows, int box_cols) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols * 2)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t es[2] = {1, 1};
    EncodeFn fn = encode_fn();
    if (!fn) throw_unsupported("cuTensorMapEncodeTiled unavailable");
    const CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw_unsupported("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return m;
}

void run_qkv_gemm(const QkvGemmArgs& g, cudaStream_t st) {
    QkvArgs a{};
    a.M = g.batch * g.L;
    a.L = g.L;
    a.H = g.heads;
    a.dk = g.dk;
    a.dv = g.dv;
    a.npred = g.npred;
    a.n_out = g.heads * (2 * g.dk + g.dv) + g.npred;
    a.kdim = g.d_model;
    a.q = static_cast<__nv_bfloat16*>(g.q);
    a.k = static_cast<__nv_bfloat16*>(g.k);
    a.v = static_cast<__nv_bfloat16*>(g.v);
    a.r = g.r;
    const CUtensorMap mx = make_map(g.x, a.M, a.kdim, kBM, kBK);
    const CUtensorMap mw = make_map(g.w, a.n_out, a.kdim, kBN, kBK);
    a.tma_store = (g.dk % 64 == 0 && g.dv % 64 == 0 && g.L % 32 == 0) ? 1 : 0;
    // store maps: each head slab as rows of d columns, [32 rows][64 cols] boxes
    const CUtensorMap mq = a.tma_store ? make_map(g.q, g.batch * g.heads * g.L, g.dk, 32, 64) : mx;
    const CUtensorMap mk = a.tma_store ? make_map(g.k, g.batch * g.heads * g.L, g.dk, 32, 64) : mx;
    const CUtensorMap mv = a.tma_store ? make_map(g.v, g.batch * g.heads * g.L, g.dv, 32, 64) : mx;
    const int sms = sm_count();
    const int64_t ntiles = ceil_div_i(a.M, kBM) * ceil_div_i(a.n_out, kBN);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ntiles, sms));
    cudaFuncSetAttribute(qkv_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    qkv_gemm_kernel<<<grid, kThreads, kSmem, st>>>(mx, mw, mq, mk, mv, a);
    note_launch();
}

}  // namespace dsa
