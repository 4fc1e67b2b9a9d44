// Microbenchmark: the L2 -> SM fabric ceiling on this GPU for the attention
// kernels' access pattern -- 128-byte rows gathered from an L2-resident
// buffer (64 MB, warmed), L1 bypassed (ld.global.cg), 8 lanes per row,
// U independent 16-byte loads in flight per lane, all SMs busy.  Variants:
//   rows at random (the gather), rows in sequence (a streaming read),
//   and TMA bulk copies of 128-byte rows into shared memory (cp.async.bulk).
// Prints GB/s and bytes per SM clock chip-wide (at the current SM clock).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_fabric_bin tools/l2_fabric_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int kRowB = 128;
constexpr int64_t kRows = 64ll * 1024 * 1024 / kRowB;  // 64 MB

__device__ __forceinline__ uint4 ldcg(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <int U, bool RANDOM>
__global__ void __launch_bounds__(256) gather_rows(const uint4* __restrict__ buf, int iters, uint4* sink) {
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    uint4 acc = make_uint4(0, 0, 0, 0);
    uint64_t state = 0x9E3779B97F4A7C15ull * static_cast<uint64_t>(gwarp * 4 + (lane >> 3) + 1);
    int64_t seq = (gwarp * 4 + (lane >> 3)) * 977;
    for (int it = 0; it < iters; ++it) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int64_t row;
            if (RANDOM) {
                state = state * 6364136223846793005ull + 1442695040888963407ull;
                row = static_cast<int64_t>((state >> 33) % static_cast<uint64_t>(kRows));
            } else {
                row = (seq++) % kRows;
            }
            x[u] = ldcg(buf + row * 8 + (lane & 7));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc.x ^= x[u].x; acc.y ^= x[u].y; acc.z ^= x[u].z; acc.w ^= x[u].w;
        }
    }
    if (acc.x == 0x12345678u && acc.y == 0x9abcdef0u) sink[0] = acc;
}

template <class K>
static void run(const char* name, K kern, const uint4* buf, uint4* sink, int ctas, int iters, int U, double clk_ghz) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<ctas, 256>>>(buf, 4, sink);  // warm
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    kern<<<ctas, 256>>>(buf, iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = static_cast<double>(ctas) * 256 * iters * U * 16;
    std::printf("%-34s %8.1f GB/s  %7.0f B/clk chip-wide (at %.3f GHz)  %.3f ms\n", name, bytes / ms * 1e-6,
                bytes / (ms * 1e-3) / (clk_ghz * 1e9), clk_ghz, ms);
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double ghz = clk_khz * 1e-6;
    uint4* buf;
    uint4* sink;
    cudaMalloc(&buf, kRows * kRowB);
    cudaMalloc(&sink, 64);
    cudaMemset(buf, 1, kRows * kRowB);
    const int sms = prop.multiProcessorCount;
    std::printf("%s, %d SMs, max SM clock %.3f GHz, L2 %d MB, buffer 64 MB\n", prop.name, sms, ghz, prop.l2CacheSize >> 20);
    for (int cps : {4, 8}) {
        const int ctas = sms * cps;
        std::printf("-- %d CTAs of 256 threads per SM\n", cps);
        run("random rows, 4 loads in flight", gather_rows<4, true>, buf, sink, ctas, 2000, 4, ghz);
        run("random rows, 8 loads in flight", gather_rows<8, true>, buf, sink, ctas, 1000, 8, ghz);
        run("random rows, 16 loads in flight", gather_rows<16, true>, buf, sink, ctas, 500, 16, ghz);
        run("sequential rows, 8 in flight", gather_rows<8, false>, buf, sink, ctas, 1000, 8, ghz);
        run("sequential rows, 16 in flight", gather_rows<16, false>, buf, sink, ctas, 500, 16, ghz);
    }
    return 0;
}
