// The band attention core shared by the attention kernels and the fused
// select + attention kernel: one warp, up to 8 query rows (one per MMA
// column), a stream of gathered keys in 32-key chunks.  S^T = K_chunk .
// Q^T with mma.sync m16n8k16 (K fragments straight from global memory,
// the d order permuted so each lane's fragment is one 16-byte load), online
// softmax in fp32 (log2 domain), Z^T += V_chunk^T . P^T with V rows by
// 16-byte cp.async into XOR-swizzled shared memory (ldmatrix.trans); key
// indices run two chunks ahead of their gathers.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace dsa {
namespace bc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    const int n = valid ? 16 : 0;  // src-size 0 -> zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// 2^x on the SFU (ex2.approx.ftz: -inf -> +0); softmax weights are rounded
// to bf16 before use, far coarser than its ~2^-22 relative error
__device__ __forceinline__ float fast_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

// 8 x 8 b16 transpose across the warp: the lane holding row lane/4, columns
// 2 (lane%4), +1 gets row lane/4, columns 2 (lane%4), +1 of the TRANSPOSE --
// turns an m16n8 accumulator half (keys x queries) into the k16n8 B-fragment
// half (P^T[keys 2c4, 2c4+1][query g]) without a shared-memory round trip.
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
    uint32_t r;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(r) : "r"(x));
    return r;
}

// Row r of a [rows][D] bf16 tile, 16-byte chunk c, XOR-swizzled within 8 chunks.
template <int D>
__device__ __forceinline__ uint32_t swz(int r, int c) {
    constexpr int kChunks = D / 8;  // 16-byte chunks per row
    return static_cast<uint32_t>(r * D * 2 + (((c & 7) ^ (r & 7)) | (c & ~7)) * 16);
    (void)kChunks;
}

// Per-warp shared memory: the double-buffered V rows of a 32-key chunk; the
// Z rows are staged in v[0] once the key loop is done.  8 KB (d = 64) per
// warp, 128 KB per 16-warp CTA: the rest of the SM's 256 KB stays L1, which
// the K-row gathers hit 20-26 % of the time (a third V stage -- 213 KB per
// CTA -- measured SLOWER: C1 0.51 -> 0.64 ms, C4 24.3 -> 30.7 ms).
template <int D>
struct BandSmemV2 {
    __nv_bfloat16 v[2][32 * D];
};

template <int D>
__device__ __forceinline__ void load_k_frag(const __nv_bfloat16* __restrict__ Kp, uint32_t idx,
                                            int g, int c4, uint4 (&kw)[2][2][D / 64 * 2]) {
    // two m-tiles x rows (g, g+8): this lane's D/4 elements are the 16-byte
    // pieces [32 v + 8 c4, +8): one load instruction covers 64 contiguous
    // bytes of each row (full 32-byte sectors)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t j = __shfl_sync(0xffffffffu, idx, mt * 16 + g + h * 8);
            const uint4* src = reinterpret_cast<const uint4*>(Kp + static_cast<int64_t>(j) * D + c4 * 8);
#pragma unroll
            for (int v = 0; v < D / 32; ++v) kw[mt][h][v] = __ldg(src + v * 4);
        }
}

// kRows query rows r0.. (MMA columns); SEG: column c only sees stream keys in
// [sb(c), sb(c+1)) (this thread's two columns: [sb0, sb1), [sb1, sb2)).
// chunk_idx(ch) returns this lane's key index of chunk ch (lane = row).
template <int D, int kRows, bool SEG, class IdxFn>
__device__ __forceinline__ void band_core(BandSmemV2<D>& sm, const __nv_bfloat16* __restrict__ Q,
                                          const __nv_bfloat16* __restrict__ Kp, const __nv_bfloat16* __restrict__ Vp,
                                          int64_t pair, int64_t L, int64_t r0, int64_t nkeys, int64_t sb0,
                                          int64_t sb1, int64_t sb2, int scale, __nv_bfloat16* __restrict__ Z,
                                          IdxFn chunk_idx, int lane) {
    constexpr int CH = 32;
    constexpr int NW = D / 32;  // uint4 per lane per K row segment (D/4 bf16)
    const int g = lane >> 2, c4 = lane & 3;
    constexpr int kChunks16 = D / 8;

    // Q^T B-fragments (same d permutation as K): row g, pieces [32 v + 8 c4, +8)
    uint32_t qw[D / 8];
    {
        const bool ok = g < kRows && r0 + g < L;
        const uint4* src = reinterpret_cast<const uint4*>(Q + (pair * L + (ok ? r0 + g : 0)) * D + c4 * 8);
#pragma unroll
        for (int v = 0; v < NW; ++v) {
            const uint4 x = ok ? __ldg(src + v * 4) : make_uint4(0, 0, 0, 0);
            qw[4 * v + 0] = x.x;
            qw[4 * v + 1] = x.y;
            qw[4 * v + 2] = x.z;
            qw[4 * v + 3] = x.w;
        }
    }
    const int nchunks = static_cast<int>((nkeys + CH - 1) / CH);
    // V rows of one chunk: lane owns 16-byte column chunk c of rows rl, rl + RPI, ..
    // (the swizzle and row offsets fold to constants per unrolled step)
    auto load_v = [&](int buf, uint32_t idx, int ch) {
        constexpr int RPI = 32 / kChunks16;  // rows per step
        const int c = lane % kChunks16, rl = lane / kChunks16;
        const uint32_t vb = smem_u32(sm.v[buf]);
        const bool full = static_cast<int64_t>(ch + 1) * CH <= nkeys;
        const int left = static_cast<int>(nkeys - static_cast<int64_t>(ch) * CH);
#pragma unroll
        for (int i = 0; i < CH / RPI; ++i) {
            const int r = rl + i * RPI;
            const uint32_t j = __shfl_sync(0xffffffffu, idx, r);
            cp_async16(vb + swz<D>(r, c), Vp + static_cast<size_t>(j) * D + c * 8, full || r < left);
        }
    };
    // indices run two chunks ahead, so chunk c+1's K/V loads never wait on
    // its index load
    const uint32_t idx0 = chunk_idx(0);
    uint32_t idx_n = nchunks > 1 ? chunk_idx(1) : 0u;
    uint4 kw[2][2][NW];
    load_k_frag<D>(Kp, idx0, g, c4, kw);
    load_v(0, idx0, 0);
    cp_async_commit();

    const float sl2 = (scale ? rsqrtf(static_cast<float>(D)) : 1.f) * 1.4426950408889634f;
    float m_run[2] = {-INFINITY, -INFINITY};
    float l_part[2] = {0.f, 0.f};
    float zacc[D / 16][4];
#pragma unroll
    for (int t = 0; t < D / 16; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) zacc[t][u] = 0.f;

    for (int ch = 0; ch < nchunks; ++ch) {
        const int buf = ch & 1;
        // prefetch the next chunk: indices, K fragments (registers), V (cp.async)
        uint4 kn[2][2][NW];
        const uint32_t idx_nn = ch + 2 < nchunks ? chunk_idx(ch + 2) : 0u;
        if (ch + 1 < nchunks) {
            load_k_frag<D>(Kp, idx_n, g, c4, kn);
            load_v(buf ^ 1, idx_n, ch + 1);
        }
        idx_n = idx_nn;
        cp_async_commit();
        // ---- S^T = K_chunk . Q^T (2 m-tiles of 16 keys)
        float s[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
            for (int u = 0; u < 4; ++u) s[mt][u] = 0.f;
            const uint32_t* ka = reinterpret_cast<const uint32_t*>(kw[mt][0]);
            const uint32_t* kb = reinterpret_cast<const uint32_t*>(kw[mt][1]);
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks)
                mma16816(s[mt], ka[2 * ks], kb[2 * ks], ka[2 * ks + 1], kb[2 * ks + 1], qw[2 * ks], qw[2 * ks + 1]);
        }
        // ---- online softmax over keys
        const int base = ch * CH;
        float cmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int key = base + mt * 16 + g + (u >> 1) * 8;
                bool live = key < nkeys;
                if (SEG) live = (u & 1) ? (key >= sb1 && key < sb2) : (key >= sb0 && key < sb1);
                const float x = live ? s[mt][u] * sl2 : -INFINITY;
                s[mt][u] = x;
                cmax[u & 1] = fmaxf(cmax[u & 1], x);
            }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 4));
            cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 8));
            cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 16));
        }
        float corr[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float mn = fmaxf(m_run[h], cmax[h]);
            corr[h] = m_run[h] == -INFINITY ? 0.f : fast_ex2(m_run[h] - mn);
            m_run[h] = mn;
            l_part[h] *= corr[h];
        }
#pragma unroll
        for (int t = 0; t < D / 16; ++t) {
            zacc[t][0] *= corr[0];
            zacc[t][1] *= corr[1];
            zacc[t][2] *= corr[0];
            zacc[t][3] *= corr[1];
        }
        // P^T as MMA B fragments straight from the S^T accumulators: bf16 pairs
        // (key g / g + 8, queries 2 c4, 2 c4 + 1) transposed across the warp
        uint32_t pb[2][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            float pv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                // a column may have no live key yet (m_run = -inf): weight 0
                pv[u] = (SEG && s[mt][u] == -INFINITY) ? 0.f : fast_ex2(s[mt][u] - m_run[u & 1]);
                // the weight the MMA sees is the bf16 value; the row sum keeps fp32 (as before)
                l_part[u & 1] += pv[u];
            }
            pb[mt][0] = movm_t(pack_bf16(pv[0], pv[1]));
            pb[mt][1] = movm_t(pack_bf16(pv[2], pv[3]));
        }
        cp_async_wait<1>();
        __syncwarp();
        // ---- Z^T += V_chunk^T . P^T
        const uint32_t vb = smem_u32(sm.v[buf]);
#pragma unroll
        for (int ks = 0; ks < CH / 16; ++ks) {
            const uint32_t b0 = pb[ks][0], b1 = pb[ks][1];
#pragma unroll
            for (int mt = 0; mt < D / 16; ++mt) {
                const int mi = lane >> 3;
                const int row = ks * 16 + (mi >> 1) * 8 + (lane & 7);
                const int chk = mt * 2 + (mi & 1);
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(vb + swz<D>(row, chk), a0, a1, a2, a3);
                mma16816(zacc[mt], a0, a1, a2, a3, b0, b1);
            }
        }
        __syncwarp();
        if (ch + 1 < nchunks) {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int v = 0; v < NW; ++v) kw[mt][h][v] = kn[mt][h][v];
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        l_part[h] += __shfl_xor_sync(0xffffffffu, l_part[h], 4);
        l_part[h] += __shfl_xor_sync(0xffffffffu, l_part[h], 8);
        l_part[h] += __shfl_xor_sync(0xffffffffu, l_part[h], 16);
    }
    __syncwarp();  // every lane done with the V buffers: v[0] now stages Z
    __nv_bfloat16* zst = sm.v[0];
    const float inv0 = l_part[0] > 0.f ? 1.f / l_part[0] : 0.f;
    const float inv1 = l_part[1] > 0.f ? 1.f / l_part[1] : 0.f;
#pragma unroll
    for (int mt = 0; mt < D / 16; ++mt) {
        const int d0 = mt * 16 + g;
        zst[(2 * c4) * D + d0] = __float2bfloat16_rn(zacc[mt][0] * inv0);
        zst[(2 * c4 + 1) * D + d0] = __float2bfloat16_rn(zacc[mt][1] * inv1);
        zst[(2 * c4) * D + d0 + 8] = __float2bfloat16_rn(zacc[mt][2] * inv0);
        zst[(2 * c4 + 1) * D + d0 + 8] = __float2bfloat16_rn(zacc[mt][3] * inv1);
    }
    __syncwarp();
    for (int t = lane; t < kRows * kChunks16; t += 32) {
        const int r = t / kChunks16, c = t % kChunks16;
        if (r0 + r < L)
            *reinterpret_cast<uint4*>(Z + (pair * L + r0 + r) * D + c * 8) =
                *reinterpret_cast<const uint4*>(&zst[r * D + c * 8]);
    }
}

}  // namespace bc
}  // namespace dsa
