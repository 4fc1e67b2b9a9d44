// Microbenchmark: gathering 128-byte K and V rows by index lists, the access
// pattern of the C2 band attention (128 pairs x 4096 rows, 512 bands of 205
// sorted random keys per pair, one warp per band, 8 bands per CTA).  Compares
//   0: LDG.128 straight into registers (8 lanes per row),
//   1: cp.async 16 B into shared memory, then LDS,
//   2: TMA tile::gather4 (4 rows per instruction, one lane issues) into
//      shared memory with an mbarrier, then LDS.
// Prints gathered GB/s (K + V row bytes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench tools/gather_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

constexpr int kPairs = 128, kL = 4096, kD = 64, kBands = 512, kKeep = 205, kChunk = 16;
constexpr int kRowB = kD * 2;  // 128 bytes

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(256) gather_ldg(const uint4* __restrict__ K, const uint4* __restrict__ V,
                                                  const int* __restrict__ idx, uint4* sink) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = blockIdx.y, band = blockIdx.x * 8 + warp;
    const int* lst = idx + (static_cast<int64_t>(pair) * kBands + band) * kKeep;
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int c0 = 0; c0 < kKeep; c0 += kChunk) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int e = c0 + i * 4 + (lane >> 3);
            if (e < kKeep) {
                const int64_t row = static_cast<int64_t>(pair) * kL + __ldg(lst + e);
                const uint4 a = __ldg(K + row * 8 + (lane & 7));
                const uint4 b = __ldg(V + row * 8 + (lane & 7));
                acc.x ^= a.x ^ b.x; acc.y ^= a.y ^ b.y; acc.z ^= a.z ^ b.z; acc.w ^= a.w ^ b.w;
            }
        }
    }
    if (acc.x == 0x12345678u) sink[0] = acc;
}

__global__ void __launch_bounds__(256) gather_cpasync(const uint4* __restrict__ K, const uint4* __restrict__ V,
                                                      const int* __restrict__ idx, uint4* sink) {
    extern __shared__ __align__(1024) uint4 dyn[];  // [8 warps][2 stages][K + V rows]
    auto buf = reinterpret_cast<uint4 (*)[2][2 * kChunk * 8]>(dyn);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = blockIdx.y, band = blockIdx.x * 8 + warp;
    const int* lst = idx + (static_cast<int64_t>(pair) * kBands + band) * kKeep;
    uint4 acc = make_uint4(0, 0, 0, 0);
    auto issue = [&](int c0, int st) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = i * 4 + (lane >> 3), e = c0 + r;
            const bool ok = e < kKeep;
            const int64_t row = static_cast<int64_t>(pair) * kL + (ok ? __ldg(lst + e) : 0);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(&buf[warp][st][r * 8 + (lane & 7)])),
                         "l"(K + row * 8 + (lane & 7)), "r"(ok ? 16 : 0));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(&buf[warp][st][(kChunk + r) * 8 + (lane & 7)])),
                         "l"(V + row * 8 + (lane & 7)), "r"(ok ? 16 : 0));
        }
        asm volatile("cp.async.commit_group;\n");
    };
    issue(0, 0);
    int st = 0;
    for (int c0 = 0; c0 < kKeep; c0 += kChunk, st ^= 1) {
        if (c0 + kChunk < kKeep) issue(c0 + kChunk, st ^ 1);
        else asm volatile("cp.async.commit_group;\n");
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint4 a = buf[warp][st][i * 32 + lane];
            acc.x ^= a.x; acc.y ^= a.y; acc.z ^= a.z; acc.w ^= a.w;
        }
        __syncwarp();
    }
    if (acc.x == 0x12345678u) sink[0] = acc;
}

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* map, int r0, int r1, int r2, int r3,
                                        uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];\n" ::"r"(dst),
        "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
        : "memory");
}

__global__ void __launch_bounds__(256) gather_tma(const __grid_constant__ CUtensorMap mk,
                                                  const __grid_constant__ CUtensorMap mv, const int* __restrict__ idx,
                                                  uint4* sink) {
    extern __shared__ __align__(1024) uint4 dyn[];
    auto buf = reinterpret_cast<uint4 (*)[2][2 * kChunk * 8]>(dyn);
    __shared__ __align__(8) uint64_t bars[8][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = blockIdx.y, band = blockIdx.x * 8 + warp;
    const int* lst = idx + (static_cast<int64_t>(pair) * kBands + band) * kKeep;
    if (lane == 0) {
        for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bars[warp][s])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    uint4 acc = make_uint4(0, 0, 0, 0);
    auto issue = [&](int c0, int st) {
        // lane j < 16 holds the chunk's row j
        const int e = c0 + (lane & 15);
        const int row = pair * kL + (e < kKeep ? __ldg(lst + e) : 0);
        int r[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) r[j] = __shfl_sync(0xffffffffu, row, j);
        if (lane == 0) {
            const uint32_t b = smem_u32(&bars[warp][st]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(2 * kChunk * kRowB) : "memory");
            const uint32_t d = smem_u32(&buf[warp][st][0]);
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                gather4(d + g * 4 * kRowB, &mk, r[4 * g], r[4 * g + 1], r[4 * g + 2], r[4 * g + 3], b);
                gather4(d + (kChunk + g * 4) * kRowB, &mv, r[4 * g], r[4 * g + 1], r[4 * g + 2], r[4 * g + 3], b);
            }
        }
    };
    issue(0, 0);
    int st = 0;
    uint32_t ph[2] = {0, 0};
    for (int c0 = 0; c0 < kKeep; c0 += kChunk, st ^= 1) {
        if (c0 + kChunk < kKeep) issue(c0 + kChunk, st ^ 1);
        const uint32_t b = smem_u32(&bars[warp][st]);
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "W_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}\n" ::"r"(b),
            "r"(ph[st])
            : "memory");
        ph[st] ^= 1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint4 a = buf[warp][st][i * 32 + lane];
            acc.x ^= a.x; acc.y ^= a.y; acc.z ^= a.z; acc.w ^= a.w;
        }
        __syncwarp();
    }
    if (acc.x == 0x12345678u) sink[0] = acc;
}

int main() {
    const size_t rows = static_cast<size_t>(kPairs) * kL;
    uint4 *K, *V, *sink;
    int* idx;
    cudaMalloc(&K, rows * kRowB);
    cudaMalloc(&V, rows * kRowB);
    cudaMalloc(&sink, 64);
    cudaMemset(K, 1, rows * kRowB);
    cudaMemset(V, 2, rows * kRowB);
    std::vector<int> h(static_cast<size_t>(kPairs) * kBands * kKeep);
    std::mt19937 rng(7);
    std::vector<int> perm(kL);
    for (size_t b = 0; b < static_cast<size_t>(kPairs) * kBands; ++b) {
        for (int i = 0; i < kL; ++i) perm[i] = i;
        for (int i = 0; i < kKeep; ++i) std::swap(perm[i], perm[i + rng() % (kL - i)]);
        std::sort(perm.begin(), perm.begin() + kKeep);
        std::copy(perm.begin(), perm.begin() + kKeep, h.begin() + b * kKeep);
    }
    cudaMalloc(&idx, h.size() * 4);
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);

    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    CUtensorMap mk, mv;
    cuuint64_t dims[2] = {kD, rows};
    cuuint64_t strides[1] = {kRowB};
    cuuint32_t box[2] = {kD, 1};
    cuuint32_t es[2] = {1, 1};
    for (int t = 0; t < 2; ++t) {
        CUresult r = enc(t ? &mv : &mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, t ? static_cast<void*>(V) : static_cast<void*>(K),
                         dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("encode failed %d\n", static_cast<int>(r));
            return 1;
        }
    }
    const dim3 grid(kBands / 8, kPairs);
    const int smem = 8 * 2 * 2 * kChunk * kRowB;
    cudaFuncSetAttribute(gather_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gather_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const double bytes = static_cast<double>(kPairs) * kBands * kKeep * 2 * kRowB;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int m = 0; m < 3; ++m) {
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(e0);
            if (m == 0) gather_ldg<<<grid, 256>>>(K, V, idx, sink);
            if (m == 1) gather_cpasync<<<grid, 256, smem>>>(K, V, idx, sink);
            if (m == 2) gather_tma<<<grid, 256, smem>>>(mk, mv, idx, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0) best = std::min(best, ms);
        }
        cudaError_t err = cudaGetLastError();
        printf("method %d (%s): %.3f ms, %.0f GB/s gathered  [%s]\n", m, m == 0 ? "ldg" : m == 1 ? "cp.async" : "tma gather4",
               best, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(err));
    }
    return 0;
}
