// Phase 3: SDDMM -> sparse row softmax -> SpMM over a predicted mask
// (P/src/sparse.cpp:38-91), as one pass per query row with an online
// softmax (running max / sum rescaling) so kept scores never touch HBM.
//
// Generic CUDA-core kernel, one warp per query row: for each chunk of 32
// kept keys a lane computes one full <q, k_j> (K row gathered with 16-byte
// vector loads), the warp agrees on the running max, then every lane
// accumulates its slice of d for the chunk's V rows (coalesced row reads).
// Covers every mask layout (row lists, band lists, block lists, CSR).
// The tensor-core kernels (attention_tc.cu) take over structured masks.
#include <cuda_bf16.h>

#include "device_common.cuh"
#include "kernels.h"
#include "mask_layout.cuh"

namespace dsa {
namespace {

constexpr int kWarpsPerCta = 4;

template <class T, int D>
__device__ __forceinline__ float dot_row(const float* qs, const T* __restrict__ krow) {
    constexpr int kVec = 16 / sizeof(T);
    const uint4* src = reinterpret_cast<const uint4*>(krow);
    float acc = 0.f;
#pragma unroll
    for (int t0 = 0; t0 < D; t0 += kVec) {
        uint4 raw = __ldg(src + t0 / kVec);
        const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int u = 0; u < kVec; ++u) acc = fmaf(qs[t0 + u], to_float(e[u]), acc);
    }
    return acc;
}

// <q_seg, k_seg> over D/4 consecutive elements (16-byte loads when possible)
template <class T, int D>
__device__ __forceinline__ float dot_seg(const float (&qr)[D / 4], const T* __restrict__ kseg) {
    constexpr int N = D / 4;
    constexpr int kBytes = N * static_cast<int>(sizeof(T));
    float acc = 0.f;
    if constexpr (kBytes % 16 == 0) {
        constexpr int kVec = 16 / sizeof(T);
        const uint4* src = reinterpret_cast<const uint4*>(kseg);
        uint4 raw[kBytes / 16];
#pragma unroll
        for (int v = 0; v < kBytes / 16; ++v) raw[v] = __ldg(src + v);
#pragma unroll
        for (int v = 0; v < kBytes / 16; ++v) {
            const T* e = reinterpret_cast<const T*>(&raw[v]);
#pragma unroll
            for (int u = 0; u < kVec; ++u) acc = fmaf(qr[v * kVec + u], to_float(e[u]), acc);
        }
    } else {
#pragma unroll
        for (int u = 0; u < N; ++u) acc = fmaf(qr[u], to_float(kseg[u]), acc);
    }
    return acc;
}

// kPer consecutive elements of a row as floats with one vector load
template <class T, int N>
__device__ __forceinline__ void load_vec(const T* __restrict__ src, float (&out)[N]) {
    constexpr int kBytes = N * static_cast<int>(sizeof(T));
    if constexpr (kBytes == 16) {
        const uint4 r = __ldg(reinterpret_cast<const uint4*>(src));
        const T* e = reinterpret_cast<const T*>(&r);
#pragma unroll
        for (int u = 0; u < N; ++u) out[u] = to_float(e[u]);
    } else if constexpr (kBytes == 8) {
        const uint2 r = __ldg(reinterpret_cast<const uint2*>(src));
        const T* e = reinterpret_cast<const T*>(&r);
#pragma unroll
        for (int u = 0; u < N; ++u) out[u] = to_float(e[u]);
    } else if constexpr (kBytes == 4) {
        const uint32_t r = __ldg(reinterpret_cast<const unsigned int*>(src));
        const T* e = reinterpret_cast<const T*>(&r);
#pragma unroll
        for (int u = 0; u < N; ++u) out[u] = to_float(e[u]);
    } else {
#pragma unroll
        for (int u = 0; u < N; ++u) out[u] = to_float(src[u]);
    }
}

// One warp per query row.  Scores: lane = kept key (its K row in 16-byte
// loads).  Output: lane = kPer CONSECUTIVE dims, so a V row is one
// coalesced warp-wide vector read; the 32 keys of a chunk are unrolled in
// groups of 8 so eight independent V gathers are in flight per lane.
template <class T, int D>
__global__ void __launch_bounds__(kWarpsPerCta * 32) attn_rows_generic(AttnArgs a) {
    constexpr int kPer = D >= 32 ? D / 32 : 1;  // output dims per lane
    constexpr int kLanes = D / kPer;            // lanes holding output dims
    __shared__ float qs[kWarpsPerCta][D];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row_global = static_cast<int64_t>(blockIdx.x) * kWarpsPerCta + warp;
    if (row_global >= a.pairs * a.L) return;
    const int64_t pair = row_global / a.L, i = row_global % a.L;
    const T* q = static_cast<const T*>(a.q) + (pair * a.L + i) * D;
    const T* kb = static_cast<const T*>(a.k) + pair * a.L * D;
    const T* vb = static_cast<const T*>(a.v) + pair * a.L * D;
    const float sc = a.scale ? rsqrtf(static_cast<float>(D)) : 1.f;
    for (int c = lane; c < D; c += 32) qs[warp][c] = to_float(q[c]) * sc;
    __syncwarp();
    const RowList rl = row_list(a, pair, i);
    const int total = rl.count * rl.expand;
    const int dl = lane < kLanes ? lane * kPer : 0;  // this lane's first output dim
    float qr[D / 4];  // this lane's quarter of q (score segment)
#pragma unroll
    for (int u = 0; u < D / 4; ++u) qr[u] = qs[warp][(lane & 3) * (D / 4) + u];
    float m = -INFINITY, l = 0.f, acc[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) acc[u] = 0.f;
    for (int p0 = 0; p0 < total; p0 += 32) {
        const int p = p0 + lane;
        int j = -1;
        if (p < total) {
            j = rl.expand == 1 ? static_cast<int>(rl.cols[p])
                               : static_cast<int>(rl.cols[p / rl.expand]) * rl.expand + p % rl.expand;
            if (j >= a.L) j = -1;  // ragged last block
        }
        // scores: four lanes per key (each a D/4 segment, 2 x 16 B for bf16
        // D = 64), eight keys per round -> a K row is one L1 wavefront per
        // 4 lanes instead of one per lane; reduce the quarter sums, then move
        // key t's score to lane t
        float s = -INFINITY;
        const int nval = min(32, total - p0);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r * 8 >= nval) break;
            const int jr = __shfl_sync(0xffffffffu, j, r * 8 + (lane >> 2));
            float part = 0.f;
            if (jr >= 0) part = dot_seg<T, D>(qr, kb + static_cast<int64_t>(jr) * D + (lane & 3) * (D / 4));
            part += __shfl_xor_sync(0xffffffffu, part, 1);
            part += __shfl_xor_sync(0xffffffffu, part, 2);
            const float got = __shfl_sync(0xffffffffu, part, 4 * (lane & 7));
            if ((lane >> 3) == r) s = got;
        }
        if (j < 0) s = -INFINITY;
        const float mnew = fmaxf(m, warp_max(s));
        const float w = j >= 0 ? expf(s - mnew) : 0.f;
        const float corr = m == -INFINITY ? 0.f : expf(m - mnew);
        l = l * corr + warp_sum(w);
#pragma unroll
        for (int u = 0; u < kPer; ++u) acc[u] *= corr;
        m = mnew;
        const int jj = j >= 0 ? j : 0;  // dropped keys gather row 0 with weight 0
        for (int t0 = 0; t0 < nval; t0 += 8) {
            float vv[8][kPer], wt[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                wt[t] = __shfl_sync(0xffffffffu, w, t0 + t);
                const int jt = __shfl_sync(0xffffffffu, jj, t0 + t);
                load_vec<T, kPer>(vb + static_cast<int64_t>(jt) * D + dl, vv[t]);
            }
#pragma unroll
            for (int t = 0; t < 8; ++t)
#pragma unroll
                for (int u = 0; u < kPer; ++u) acc[u] = fmaf(wt[t], vv[t][u], acc[u]);
        }
    }
    T* z = static_cast<T*>(a.z) + (pair * a.L + i) * D;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    if (lane < kLanes) {
#pragma unroll
        for (int u = 0; u < kPer; ++u) z[dl + u] = from_float<T>(acc[u] * inv);
    }
    if (lane == 0 && a.empty_rows) a.empty_rows[pair * a.L + i] = (l > 0.f) ? 0 : 1;
}

template <class T>
void dispatch(const AttnArgs& a, cudaStream_t st) {
    const unsigned grid = static_cast<unsigned>(ceil_div_i(a.pairs * a.L, kWarpsPerCta));
    switch (a.D) {
        case 16: attn_rows_generic<T, 16><<<grid, kWarpsPerCta * 32, 0, st>>>(a); break;
        case 32: attn_rows_generic<T, 32><<<grid, kWarpsPerCta * 32, 0, st>>>(a); break;
        case 64: attn_rows_generic<T, 64><<<grid, kWarpsPerCta * 32, 0, st>>>(a); break;
        case 128: attn_rows_generic<T, 128><<<grid, kWarpsPerCta * 32, 0, st>>>(a); break;
        default: throw_unsupported("head dim d must be one of 16, 32, 64, 128");
    }
}

}  // namespace

void run_attention(const AttnArgs& a, cudaStream_t st) {
    if (block_tc_supported(a)) {
        run_block_tc(a, st);
        return;
    }
    if (band_attention_supported(a)) {
        run_band_attention(a, st);
        return;
    }
    if (a.bf16) dispatch<__nv_bfloat16>(a, st);
    else dispatch<float>(a, st);
    note_launch();
}

}  // namespace dsa
