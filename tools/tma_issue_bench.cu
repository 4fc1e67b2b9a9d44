// Microbenchmark: cp.async.bulk (global -> shared, L2-resident source) issue
// cost and per-SM throughput, by copy size and number of issuing warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2110_11299_b200/csrc -o tma_issue_bench tools/tma_issue_bench.cu
#include <cstdio>
#include <cstdint>
#include "tc_sm100.cuh"

using namespace dsa;

__global__ void bench(const unsigned char* src, int bytes, int copies, int issuers, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar[8][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { for (int i = 0; i < 16; ++i) tc::mbar_init(&bar[i / 2][i % 2], 1); tc::fence_barrier_init(); }
    __syncthreads();
    if (warp < issuers && lane == 0) {
        const uint32_t dst0 = tc::smem_addr(sm) + warp * 2 * bytes;
        long long t0 = clock64(), issue = 0;
        for (int c = 0; c < copies; ++c) {
            const int s = c & 1;
            if (c >= 2) tc::mbar_wait(&bar[warp][s], ((c >> 1) - 1) & 1);
            const long long ti = clock64();
            tc::mbar_expect_tx(&bar[warp][s], bytes);
            // source: a 4 MB window (L2 resident after the first pass), per block / warp offset
            const size_t off = ((size_t)(blockIdx.x * 8 + warp) * 65536 + (size_t)c * bytes) % (4u << 20);
            tc::bulk_g2s(dst0 + s * bytes, src + off, bytes, &bar[warp][s]);
            issue += clock64() - ti;
        }
        tc::mbar_wait(&bar[warp][(copies - 1) & 1], ((copies - 1) >> 1) & 1);
        const long long t1 = clock64();
        if (blockIdx.x == 0 && warp == 0) { out[0] = t1 - t0; out[1] = issue; }
    }
    __syncthreads();
}

int main() {
    unsigned char* src;
    cudaMalloc(&src, 8u << 20);
    cudaMemset(src, 1, 8u << 20);
    unsigned long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int bytes : {2048, 4096, 8192, 16384})
        for (int iss : {1, 2, 4, 8}) {
            const int copies = 512;
            const int smem = iss * 2 * bytes;
            if (smem > 200 * 1024) continue;
            bench<<<148, 256, smem>>>(src, bytes, copies, iss, d);
            bench<<<148, 256, smem>>>(src, bytes, copies, iss, d);
            unsigned long long h[2] = {0, 0};
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            const double cyc = (double)h[0] / copies;
            printf("bytes %5d issuers %d: %.0f cycles per copy per issuer, issue %.0f cyc; SM throughput %.1f B/cyc (%s)\n",
                   bytes, iss, cyc, (double)h[1] / copies, bytes * iss / cyc, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
