// Microbenchmark: cost of tcgen05.mma.kind::f16 (bf16 in, f32 accumulate,
// M = 128, K = 16 per instruction, A/B K-major in shared memory) + commit
// when issued from one thread, by MMAs per commit and by the number of
// issuing warps per CTA (each with its own TMEM columns and barriers).
// Measured r02 (B200): a commit costs its issuing thread ~800 cycles
// whatever the number of commits in flight, independent of N and of the
// operand layout; MMAs between commits ~50-60 cycles each.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2110_11299_b200/csrc -o mma_issue_bench tools/mma_issue_bench.cu
#include <cstdio>
#include <cstdint>
#include "tc_sm100.cuh"

using namespace dsa;

__global__ void bench(int N, int iters, int ksteps, int issuers, int depth, int nomma, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar[4][8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (128 * 64 + 256 * 64) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x == 0) { for (int i = 0; i < 32; ++i) tc::mbar_init(&bar[i / 8][i % 8], 1); tc::fence_barrier_init(); }
    if (warp == 0) tc::tmem_alloc<512>(&slot);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = slot;
    if (warp < issuers && lane == 0) {
        const uint32_t a_s = tc::smem_addr(sm), b_s = a_s + 128 * 64;
        const uint32_t idesc = tc::idesc_bf16_f32(128, N);
        const uint64_t ad = tc::desc_kmajor_nosw(a_s, 128 * 16, 128), bd = tc::desc_kmajor_nosw(b_s, 256 * 16, 128);
        const int cols = 512 / issuers / N;
        const uint32_t tbase = tm + warp * (512 / issuers);
        uint64_t* b = bar[warp];
        int c = 0;
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (!nomma)
                for (int k = 0; k < ksteps; ++k) tc::mma_bf16(tbase + (i % cols) * N, ad, bd, idesc, k > 0);
            if (c >= depth) tc::mbar_wait(&b[c % depth], ((c / depth) - 1) & 1);
            tc::commit(&b[c % depth]);
            ++c;
        }
        tc::mbar_wait(&b[(c - 1) % depth], ((c - 1) / depth) & 1);
        long long t1 = clock64();
        if (blockIdx.x == 0 && warp == 0) out[0] = t1 - t0;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tm);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = 128 * 64 + 256 * 64;
    struct C { int N, ks, iss, depth, nomma; };
    const C cs[] = {{64, 1, 1, 4, 1}, {64, 1, 1, 4, 0}, {64, 1, 2, 4, 0}, {64, 1, 4, 4, 0}, {64, 2, 1, 4, 0},
                    {64, 2, 2, 4, 0}, {64, 2, 4, 4, 0}, {64, 4, 4, 4, 0}, {64, 8, 4, 4, 0}, {128, 1, 4, 4, 0},
                    {128, 2, 2, 4, 0}, {64, 16, 1, 4, 0}};
    for (const C& c : cs) {
        const int iters = 1024 / c.ks;
        bench<<<148, 128, smem>>>(c.N, iters, c.ks, c.iss, c.depth, c.nomma, d);
        bench<<<148, 128, smem>>>(c.N, iters, c.ks, c.iss, c.depth, c.nomma, d);
        unsigned long long h = 0;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        const double per = (double)h / (iters * c.ks);
        printf("N=%3d mma/commit %2d issuers %d %s: %.1f cycles per MMA per issuer -> %.1f per MMA per SM (%s)\n", c.N,
               c.ks, c.iss, c.nomma ? "(commits only)" : "", per, per / c.iss, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
