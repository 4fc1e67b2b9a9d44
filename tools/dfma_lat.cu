// Microbenchmark: latency of a dependent fp64 FMA chain (the reference
// projection chain shape: 64 steps, P from shared memory), one thread.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(const double* __restrict__ p, const float* __restrict__ x, double* out, long long* cyc, int mode) {
    __shared__ double ps[64 * 16];
    for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) ps[i] = p[i];
    __syncthreads();
    if (threadIdx.x != 0) return;
    double xr[64];
    for (int t = 0; t < 64; ++t) xr[t] = x[t];
    const int j = static_cast<int>(clock() & 7);
    long long t0 = clock64();
    double acc = 0.0;
    if (mode == 0) {
#pragma unroll
        for (int t = 0; t < 64; ++t) acc = fma(xr[t], 1.0000001, acc);
    } else {
#pragma unroll
        for (int t = 0; t < 64; ++t) acc = fma(xr[t], ps[t * 16 + j], acc);
    }
    long long t1 = clock64();
    out[0] = acc;
    cyc[0] = t1 - t0;
}

int main() {
    double* p; float* x; double* o; long long* c;
    cudaMalloc(&p, 8 * 1024); cudaMalloc(&x, 4 * 64); cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    cudaMemset(p, 0, 8 * 1024); cudaMemset(x, 0, 4 * 64);
    for (int mode = 0; mode < 2; ++mode) {
        for (int r = 0; r < 3; ++r) chain<<<1, 128>>>(p, x, o, c, mode);
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("mode %d: %lld cycles for 64 dependent DFMA (%.1f per step)\n", mode, h, h / 64.0);
    }
    return 0;
}
