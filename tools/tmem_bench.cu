// Microbenchmark: tcgen05.ld 32x32b throughput (bytes / clock / SM) by warps
// per SM (measured r01: 230 B/clk at 4 warps, 340 B/clk at 8), and the
// .pack::16b variant (two 16-bit columns per register: bytes delivered to
// registers; twice as many TMEM columns per byte).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int SHAPE>
__device__ __forceinline__ void ld32(uint32_t a, uint32_t (&r)[32]) {
#define R32 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
#define OUTS "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
    if (SHAPE == 0) asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 " R32 : OUTS : "r"(a));
    if (SHAPE == 1) asm volatile("tcgen05.ld.sync.aligned.16x64b.x32.b32 " R32 : OUTS : "r"(a));
    if (SHAPE == 2) asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 " R32 : OUTS : "r"(a));
    if (SHAPE == 3) asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 " R32 : OUTS : "r"(a));
    if (SHAPE == 4) asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 " R32 : OUTS : "r"(a));
}

template <int SHAPE>
__global__ void bench(int iters, unsigned long long* out, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tm = slot;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t r0[32], r1[32];
        // pack::16b reads 64 columns per x32 instruction
        const uint32_t col = SHAPE == 4 ? (((i * 128) + (warp >> 2) * 64) & 511) : (((i * 64) + (warp >> 2) * 32) & 511);
        ld32<SHAPE>(tm + lane_base + col, r0);
        ld32<SHAPE>(tm + lane_base + ((col + 256) & 511), r1);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int x = 0; x < 32; ++x) acc ^= r0[x] + r1[x];
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
    if (acc == 0x12345678u) sink[0] = acc;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
}

template <int SHAPE>
void run(const char* name, int warps) {
    const int iters = 4096;
    unsigned long long* d;
    uint32_t* sink;
    cudaMalloc(&d, 148 * 8);
    cudaMalloc(&sink, 4);
    bench<SHAPE><<<148, warps * 32>>>(iters, d, sink);
    bench<SHAPE><<<148, warps * 32>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    // bytes delivered to registers (pack::16b: 2 columns per register)
    const double bytes = double(iters) * 2 * 32 * 32 * 4 * warps;  // per SM
    printf("%-14s warps=%2d  %7.1f B/clk/SM  (%s)\n", name, warps, bytes / avg, cudaGetErrorString(e));
    cudaFree(d);
    cudaFree(sink);
}

int main() {
    for (int w : {4, 8, 16}) {
        run<0>("32x32b.x32", w);
        run<4>("x32.pack::16b", w);
    }
    return 0;
}
