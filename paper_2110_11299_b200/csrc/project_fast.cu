// Phase 1 fast path: projection + quantisation in ONE pass over Q and K,
// with levels certified bit-identical to the reference's.
//
// The reference level is clamp(round_half_away(x64 / s)) where x64 is the
// double sequential-FMA chain of the row against P (P/src/kernels/scalar.cpp:
// 19-32) and s = max|x64| / qmax over the (b,h) tensor (P/src/predictor.cpp:
// 37-43), or per row in the per-row extension.
//
//   1. x = X . P on the fp64 tensor cores (DMMA m8n8k4, one warp per 8-row
//      group).  Any fp64 summation order satisfies |x - x64| <= 2 d 2^-53
//      |q| |p_j|, far below the fp32 storage rounding that follows;
//   2. x is kept as fp32 in shared memory with the bound
//      e = |x| 2^-23 + 1e-12 |q| |p_j|  (+ one f32 ulp when the reference
//      rounds the product through float);
//   3. amax: only elements with |x| + e >= max(|x| - e) can hold the maximum;
//      they are recomputed with the reference's own fp64 chain;
//   4. level: t = x / s is certified when it is farther than the (scaled)
//      bound from every .5 rounding boundary; the rare rest is recomputed
//      exactly.  Every emitted level equals the reference's.
//
// Per-tensor scope: a (b,h) pair is one thread-block cluster; CTAs own
// contiguous row ranges and combine the tensor max through distributed
// shared memory (atomics on rank 0), so Q and K are read from HBM once and
// only the bf16 levels are written.
#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include "device_common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace dsa {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

template <class T, int D, int KD>
__device__ __forceinline__ double exact_chain(const T* __restrict__ row, const double* pd, int j,
                                              int round_f32) {
    double acc = 0.0;
#pragma unroll 8
    for (int t = 0; t < D; ++t) acc = fma(to_double(row[t]), pd[t * KD + j], acc);
    return round_f32 ? static_cast<double>(static_cast<float>(acc)) : acc;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// One 8-row group: thread (g = lane/4, c = lane%4) owns row g, columns
// [c*D/4, (c+1)*D/4) of X (k-order permuted, which any fp64 order allows)
// and returns x[g][8*nt + 2c + {0,1}] for nt < KD/8, plus |row|^2.
template <class T, int D, int KD>
__device__ __forceinline__ void group_dmma(const T* __restrict__ row, bool valid, const double* pd,
                                           int c, int g, double (&x)[KD / 4], double& n2) {
    constexpr int KS = D / 4;  // k-steps per thread
    constexpr int kVec = 16 / sizeof(T);
    double a[KS];
    if (valid) {
        const uint4* src = reinterpret_cast<const uint4*>(row + c * KS);
#pragma unroll
        for (int v = 0; v < KS / kVec; ++v) {
            const uint4 r = __ldg(src + v);
            const T* e = reinterpret_cast<const T*>(&r);
#pragma unroll
            for (int u = 0; u < kVec; ++u) a[v * kVec + u] = to_double(e[u]);
        }
    } else {
#pragma unroll
        for (int s = 0; s < KS; ++s) a[s] = 0.0;
    }
    n2 = 0.0;
#pragma unroll
    for (int s = 0; s < KS; ++s) n2 = fma(a[s], a[s], n2);
    n2 += __shfl_xor_sync(0xffffffffu, n2, 1);
    n2 += __shfl_xor_sync(0xffffffffu, n2, 2);
#pragma unroll
    for (int nt = 0; nt < KD / 8; ++nt) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s) dmma(d0, d1, a[s], pd[(c * KS + s) * KD + nt * 8 + g]);
        x[2 * nt] = d0;
        x[2 * nt + 1] = d1;
    }
}

// The Q and K rows of one 8-row group together: the raw 16-byte loads are
// issued one group ahead (group_load) so the DMMA chains of group g overlap
// the HBM latency of group g + 1; then 2 tensors x KD/8 column tiles x 2
// k-halves = independent DMMA chains (the k split is one more fp64
// rounding, inside the bound).
template <class T, int D>
struct GroupRaw {
    static constexpr int NV = (D / 4) / (16 / static_cast<int>(sizeof(T)));
    uint4 v[2][NV];
};

template <class T, int D>
__device__ __forceinline__ void group_load(const T* __restrict__ rq, const T* __restrict__ rk, bool valid, int c,
                                           GroupRaw<T, D>& raw) {
    constexpr int KS = D / 4;
#pragma unroll
    for (int v = 0; v < GroupRaw<T, D>::NV; ++v) {
        raw.v[0][v] = valid ? __ldg(reinterpret_cast<const uint4*>(rq + c * KS) + v) : make_uint4(0, 0, 0, 0);
        raw.v[1][v] = valid ? __ldg(reinterpret_cast<const uint4*>(rk + c * KS) + v) : make_uint4(0, 0, 0, 0);
    }
}

template <class T, int D, int KD>
__device__ __forceinline__ void group_dmma2(const GroupRaw<T, D>& raw, const double* pd, int c, int g,
                                            double (&x)[2][KD / 4], double (&n2)[2]) {
    constexpr int KS = D / 4;
    constexpr int kVec = 16 / sizeof(T);
    constexpr int NV = GroupRaw<T, D>::NV;
    double a[2][KS];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const T* e = reinterpret_cast<const T*>(&raw.v[w][v]);
#pragma unroll
            for (int u = 0; u < kVec; ++u) a[w][v * kVec + u] = to_double(e[u]);
        }
        double s2 = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s) s2 = fma(a[w][s], a[w][s], s2);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
        n2[w] = s2;
    }
    double acc[2][KD / 8][2][2];
#pragma unroll
    for (int w = 0; w < 2; ++w)
#pragma unroll
        for (int nt = 0; nt < KD / 8; ++nt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) acc[w][nt][hh][0] = acc[w][nt][hh][1] = 0.0;
#pragma unroll
    for (int s = 0; s < KS / 2; ++s) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int ks = hh * (KS / 2) + s;
#pragma unroll
            for (int nt = 0; nt < KD / 8; ++nt) {
                const double b = pd[(c * KS + ks) * KD + nt * 8 + g];
                dmma(acc[0][nt][hh][0], acc[0][nt][hh][1], a[0][ks], b);
                dmma(acc[1][nt][hh][0], acc[1][nt][hh][1], a[1][ks], b);
            }
        }
    }
#pragma unroll
    for (int w = 0; w < 2; ++w)
#pragma unroll
        for (int nt = 0; nt < KD / 8; ++nt) {
            x[w][2 * nt] = acc[w][nt][0][0] + acc[w][nt][1][0];
            x[w][2 * nt + 1] = acc[w][nt][0][1] + acc[w][nt][1][1];
        }
}

__device__ __forceinline__ float bound_of(float x, float abs_e, int round_f32) {
    return fabsf(x) * (round_f32 ? 2.4e-7f : 1.2e-7f) + abs_e;
}

// Certified level, or NaN when t = x/s may sit on the other side of a .5
// rounding boundary than the reference's t (fp32 arithmetic; the margin
// covers the bound and the fp32 rounding of x * (1/s)).
__device__ __forceinline__ float certified_level(float x, float e, float inv_s, float qmax) {
    const float t = x * inv_s;
    const float at = fabsf(t);
    const float frac = at - floorf(at);
    const float margin = fmaf(at, 1e-6f, e * inv_s * 1.001f) + 1e-30f;
    if (fabsf(frac - 0.5f) <= margin) return __int_as_float(0x7fc00000);
    return fminf(fmaxf(copysignf(floorf(at + 0.5f), t), -qmax), qmax);
}

// bf16 bits of a small integer-valued float (exact: |v| <= 127)
__device__ __forceinline__ uint32_t lvl_bits(float r) { return __float_as_uint(r) >> 16; }

template <class T, int D, int KD>
__device__ __forceinline__ void stage_p(const float* __restrict__ p, double* pd, float* pn) {
    for (int i = threadIdx.x; i < D * KD; i += kThreads) pd[i] = static_cast<double>(p[i]);
    __syncthreads();
    if (threadIdx.x < KD) {
        double s2 = 0.0;
        for (int t = 0; t < D; ++t) s2 = fma(pd[t * KD + threadIdx.x], pd[t * KD + threadIdx.x], s2);
        pn[threadIdx.x] = static_cast<float>(sqrt(s2) * 1.001);
    }
}

// x (KD/4 per thread, fragment order) of one group -> levels (exact)
template <class T, int D, int KD>
__device__ __forceinline__ void quantize_group(const float* xv, float abs_e_row, const float* pn,
                                               double amax, float inv_s, double s, double qmax,
                                               const T* __restrict__ row, const double* pd, int c,
                                               int round_f32, uint16_t* __restrict__ out_pair,
                                               int64_t L, int64_t r_out, bool valid) {
    uint32_t w[KD / 8];
#pragma unroll
    for (int nt = 0; nt < KD / 8; ++nt) {
        float r[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int col = nt * 8 + 2 * c + h;
            float lv = 0.f;
            if (amax != 0.0) {
                const float x = xv[2 * nt + h];
                lv = certified_level(x, bound_of(x, abs_e_row * pn[col], round_f32), inv_s,
                                     static_cast<float>(qmax));
                if (lv != lv && valid) {  // uncertified: exact reference arithmetic
                    const double xe = exact_chain<T, D, KD>(row, pd, col, round_f32);
                    lv = static_cast<float>(fmin(fmax(round_half_away(xe / s), -qmax), qmax));
                }
            }
            r[h] = lv;
        }
        w[nt] = lvl_bits(r[0]) | (lvl_bits(r[1]) << 16);
    }
    if (valid) {
#pragma unroll
        for (int nt = 0; nt < KD / 8; ++nt)
            *reinterpret_cast<uint32_t*>(out_pair + lvl_index(L, r_out, nt * 8 + 2 * c)) = w[nt];
    }
}

// ------------------------------------------------------------ per-tensor
template <class T, int D, int KD>
__global__ void __launch_bounds__(kThreads)
    project_cluster_kernel(const T* __restrict__ q, const T* __restrict__ k,
                           const float* __restrict__ p, int64_t L, int round_f32, double qmax,
                           uint16_t* __restrict__ lq, uint16_t* __restrict__ lk,
                           double* __restrict__ sq, double* __restrict__ sk) {
    extern __shared__ __align__(16) float dyn[];
    __shared__ __align__(16) double pd[D * KD];
    __shared__ float pn[KD];
    __shared__ unsigned int lb_bits[2];        // rank 0: max(|x| - e) as float bits
    __shared__ unsigned long long am_bits[2];  // rank 0: exact amax as double bits
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned csize = cluster.num_blocks();
    const unsigned rank = cluster.block_rank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, c = lane & 3;
    const int64_t pair = blockIdx.y;
    const int64_t R = ((L + csize - 1) / csize + 7) / 8 * 8;  // rows per CTA, whole groups
    const int64_t row0 = static_cast<int64_t>(rank) * R;
    const int ngroups = static_cast<int>(R / 8);               // per tensor
    float* xs = dyn;                                           // [2*ngroups][32][KD/4]
    float* re = dyn + 2 * ngroups * 32 * (KD / 4);             // [2*ngroups][8] abs bound factors

    stage_p<T, D, KD>(p, pd, pn);
    if (tid < 2) {
        lb_bits[tid] = 0u;
        am_bits[tid] = 0ull;
    }
    cluster.sync();  // P staged; rank 0 accumulators initialised before remote atomics

    const T* base[2] = {q + pair * L * D, k + pair * L * D};
    float lb[2] = {0.f, 0.f};
    GroupRaw<T, D> nxt;
    {
        const int64_t r = row0 + warp * 8 + g;
        const bool ok = warp < ngroups && r < L;
        group_load<T, D>(base[0] + (ok ? r : 0) * D, base[1] + (ok ? r : 0) * D, ok, c, nxt);
    }
    for (int grp = warp; grp < ngroups; grp += kWarps) {
        const int64_t r = row0 + grp * 8 + g;
        const bool valid = r < L;
        const GroupRaw<T, D> cur = nxt;
        {
            const int64_t rn = r + kWarps * 8;
            const bool ok = grp + kWarps < ngroups && rn < L;
            group_load<T, D>(base[0] + (ok ? rn : 0) * D, base[1] + (ok ? rn : 0) * D, ok, c, nxt);
        }
        double x[2][KD / 4], n2[2];
        group_dmma2<T, D, KD>(cur, pd, c, g, x, n2);
#pragma unroll
        for (int w = 0; w < 2; ++w) {
            const int gi = w * ngroups + grp;
            const float abs_e = static_cast<float>(sqrt(n2[w]) * 1e-12) + 1e-30f;
            if (c == 0) re[gi * 8 + g] = abs_e;
            float* dst = xs + (static_cast<size_t>(gi) * 32 + lane) * (KD / 4);
#pragma unroll
            for (int s = 0; s < KD / 4; ++s) {
                const float xf = static_cast<float>(x[w][s]);
                dst[s] = xf;
                const int col = (s >> 1) * 8 + 2 * c + (s & 1);
                if (valid) lb[w] = fmaxf(lb[w], fabsf(xf) - bound_of(xf, abs_e * pn[col], round_f32));
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        lb[0] = fmaxf(lb[0], __shfl_xor_sync(0xffffffffu, lb[0], off));
        lb[1] = fmaxf(lb[1], __shfl_xor_sync(0xffffffffu, lb[1], off));
    }
    unsigned int* lb0 = cluster.map_shared_rank(lb_bits, 0);
    if (lane == 0) {
        atomicMax(&lb0[0], __float_as_uint(fmaxf(0.f, lb[0] * 0.999999f)));
        atomicMax(&lb0[1], __float_as_uint(fmaxf(0.f, lb[1] * 0.999999f)));
    }
    cluster.sync();
    const float LB[2] = {__uint_as_float(lb0[0]), __uint_as_float(lb0[1])};
    unsigned long long* am0 = cluster.map_shared_rank(am_bits, 0);
    for (int gi = warp; gi < 2 * ngroups; gi += kWarps) {
        const int w = gi / ngroups, grp = gi % ngroups;
        const int64_t r = row0 + grp * 8 + g;
        if (r >= L) continue;
        const float abs_e = re[gi * 8 + g];
        const float* src = xs + (static_cast<size_t>(gi) * 32 + lane) * (KD / 4);
#pragma unroll
        for (int s = 0; s < KD / 4; ++s) {
            const int col = (s >> 1) * 8 + 2 * c + (s & 1);
            const float xf = src[s];
            if (fabsf(xf) + bound_of(xf, abs_e * pn[col], round_f32) >= LB[w]) {
                const double xe = exact_chain<T, D, KD>(base[w] + r * D, pd, col, round_f32);
                atomicMax(&am0[w], static_cast<unsigned long long>(__double_as_longlong(fabs(xe))));
            }
        }
    }
    cluster.sync();
    const double amax[2] = {__longlong_as_double(static_cast<long long>(am0[0])),
                            __longlong_as_double(static_cast<long long>(am0[1]))};
    const double s[2] = {amax[0] / qmax, amax[1] / qmax};
    const float inv_s[2] = {static_cast<float>(qmax / amax[0]), static_cast<float>(qmax / amax[1])};
    uint16_t* outp[2] = {lq + pair * L * KD, lk + pair * L * KD};
    for (int gi = warp; gi < 2 * ngroups; gi += kWarps) {
        const int w = gi / ngroups, grp = gi % ngroups;
        const int64_t r = row0 + grp * 8 + g;
        const bool valid = r < L;
        quantize_group<T, D, KD>(xs + (static_cast<size_t>(gi) * 32 + lane) * (KD / 4),
                                 re[gi * 8 + g], pn, amax[w], inv_s[w], s[w], qmax,
                                 base[w] + (valid ? r : 0) * D, pd, c, round_f32,
                                 outp[w], L, valid ? r : 0, valid);
    }
    if (rank == 0 && tid < 2) (tid ? sk : sq)[pair] = amax[tid] == 0.0 ? 0.0 : s[tid];
    cluster.sync();  // rank 0's shared memory stays alive until every CTA is done with it
}

// ----------------------------------------------------------------- per-row
template <class T, int D, int KD>
__global__ void __launch_bounds__(kThreads)
    project_rows_fast_kernel(const T* __restrict__ q, const T* __restrict__ k,
                             const float* __restrict__ p, int64_t L, int round_f32, double qmax,
                             uint16_t* __restrict__ lq, uint16_t* __restrict__ lk,
                             double* __restrict__ sq, double* __restrict__ sk) {
    __shared__ __align__(16) double pd[D * KD];
    __shared__ float pn[KD];
    stage_p<T, D, KD>(p, pd, pn);
    __syncthreads();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, c = lane & 3;
    const int64_t pair = blockIdx.y;
    const int64_t ngroups = (L + 7) / 8;
    const int64_t gi = static_cast<int64_t>(blockIdx.x) * kWarps + warp;  // over 2*ngroups
    if (gi >= 2 * ngroups) return;
    const int w = static_cast<int>(gi / ngroups);
    const int64_t r = (gi % ngroups) * 8 + g;
    const bool valid = r < L;
    const T* row = (w ? k : q) + (pair * L + (valid ? r : 0)) * D;
    double x[KD / 4], n2;
    group_dmma<T, D, KD>(row, valid, pd, c, g, x, n2);
    const float abs_e = static_cast<float>(sqrt(n2) * 1e-12) + 1e-30f;
    float xf[KD / 4], lbv = 0.f;
#pragma unroll
    for (int s = 0; s < KD / 4; ++s) {
        xf[s] = static_cast<float>(x[s]);
        const int col = (s >> 1) * 8 + 2 * c + (s & 1);
        lbv = fmaxf(lbv, fabsf(xf[s]) - bound_of(xf[s], abs_e * pn[col], round_f32));
    }
    // the row's KD values live on the 4 lanes sharing g
    lbv = fmaxf(lbv, __shfl_xor_sync(0xffffffffu, lbv, 1));
    lbv = fmaxf(lbv, __shfl_xor_sync(0xffffffffu, lbv, 2));
    lbv *= 0.999999f;
    double am = 0.0;
#pragma unroll
    for (int s = 0; s < KD / 4; ++s) {
        const int col = (s >> 1) * 8 + 2 * c + (s & 1);
        if (valid && fabsf(xf[s]) + bound_of(xf[s], abs_e * pn[col], round_f32) >= lbv)
            am = fmax(am, fabs(exact_chain<T, D, KD>(row, pd, col, round_f32)));
    }
    am = fmax(am, __shfl_xor_sync(0xffffffffu, am, 1));
    am = fmax(am, __shfl_xor_sync(0xffffffffu, am, 2));
    const double s = am / qmax;
    quantize_group<T, D, KD>(xf, abs_e, pn, am, static_cast<float>(qmax / am), s, qmax, row, pd, c,
                             round_f32, (w ? lk : lq) + pair * L * KD, L, valid ? r : 0, valid);
    if (valid && c == 0) (w ? sk : sq)[pair * L + r] = am == 0.0 ? 0.0 : s;
}

int pick_cluster(int64_t L, int64_t KD) {
    // fp32 x + per-row bound factor per CTA; aim <= 96 KB, cluster <= 16
    const int64_t bytes = 2 * (L + 7 * 16) * (KD + 1) * 4;
    int c = 1;
    while (c < 16 && (bytes + c - 1) / c > 96 * 1024) c *= 2;
    return (bytes + c - 1) / c <= 150 * 1024 ? c : 0;
}

template <class T, int D, int KD>
void launch_fast(const PredictArgs& a, cudaStream_t st) {
    const T* q = static_cast<const T*>(a.q);
    const T* k = static_cast<const T*>(a.k);
    if (a.per_row) {
        const int64_t ngroups = ceil_div_i(a.L, 8);
        const dim3 grid(static_cast<unsigned>(ceil_div_i(2 * ngroups, kWarps)), static_cast<unsigned>(a.pairs));
        project_rows_fast_kernel<T, D, KD><<<grid, kThreads, 0, st>>>(q, k, a.p, a.L, a.round_f32, a.qmax,
                                                                     a.lq, a.lk, a.sq, a.sk);
        return;
    }
    const int c = pick_cluster(a.L, KD);
    const int64_t R = (ceil_div_i(a.L, c) + 7) / 8 * 8;
    const size_t smem = static_cast<size_t>(2 * (R / 8) * 32 * (KD / 4) * 4 + 2 * (R / 8) * 8 * 4);
    auto kern = project_cluster_kernel<T, D, KD>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (c > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(c), static_cast<unsigned>(a.pairs), 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(c);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, q, k, a.p, a.L, a.round_f32, a.qmax, a.lq, a.lk,
                                             a.sq, a.sk);
    if (e != cudaSuccess) throw_cuda(e, "project_cluster_kernel launch");
}

template <class T, int D>
void fast_k(const PredictArgs& a, cudaStream_t st) {
    if (a.KD == 16) launch_fast<T, D, 16>(a, st);
    else launch_fast<T, D, 32>(a, st);
}

template <class T>
void fast_d(const PredictArgs& a, cudaStream_t st) {
    switch (a.D) {
        case 32: fast_k<T, 32>(a, st); break;
        case 64: fast_k<T, 64>(a, st); break;
        default: fast_k<T, 128>(a, st); break;
    }
}

}  // namespace

bool predict_fast_supported(const PredictArgs& a) {
    if (a.KD != 16 && a.KD != 32) return false;
    if (a.D != 32 && a.D != 64 && a.D != 128) return false;  // D/4 columns per lane, 16-B loads
    if (a.D * a.KD * 8 > 40 * 1024) return false;           // static f64 P tile
    return a.per_row || pick_cluster(a.L, a.KD) > 0;
}

void run_predict_fast(const PredictArgs& a, cudaStream_t st) {
    if (a.bf16) fast_d<__nv_bfloat16>(a, st);
    else fast_d<float>(a, st);
    note_launch();
}

}  // namespace dsa
