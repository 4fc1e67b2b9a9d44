// Mask accounting on the device: prediction_accuracy
// (P/src/maskgen.cpp:94-107) between two masks of one layout --
// |pred n oracle| / |pred|, per-row counts required equal.
#include "device_common.cuh"
#include "kernels.h"
#include "mask_layout.cuh"

namespace dsa {
namespace {

constexpr int kWarps = 8;

// key t (< count * expand, clipped at L) of a row list
__device__ __forceinline__ int64_t key_at(const RowList& r, int64_t t) {
    return r.expand == 1 ? static_cast<int64_t>(r.cols[t])
                         : static_cast<int64_t>(r.cols[t / r.expand]) * r.expand + t % r.expand;
}

__device__ __forceinline__ int64_t row_keys(const RowList& r, int64_t L) {
    if (r.expand == 1) return r.count;
    int64_t n = 0;  // ragged last block: keys past L do not exist
    for (int t = 0; t < r.count; ++t) {
        const int64_t j0 = static_cast<int64_t>(r.cols[t]) * r.expand;
        n += j0 + r.expand <= L ? r.expand : (j0 < L ? L - j0 : 0);
    }
    return n;
}

// membership of key j in an ascending row list (binary search over the
// entries; BLOCK lists hold block indices)
__device__ __forceinline__ bool contains(const RowList& r, int64_t j) {
    const uint32_t v = static_cast<uint32_t>(r.expand == 1 ? j : j / r.expand);
    int lo = 0, hi = r.count;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (r.cols[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo < r.count && r.cols[lo] == v;
}

// one warp per (pair, row); out = {intersection, total, count mismatch}
__global__ void __launch_bounds__(kWarps * 32) accuracy_kernel(AttnArgs pred, AttnArgs orc,
                                                               unsigned long long* __restrict__ out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
    if (row >= pred.pairs * pred.L) return;
    const int64_t pair = row / pred.L, i = row % pred.L;
    const RowList rp = row_list(pred, pair, i), ro = row_list(orc, pair, i);
    const int64_t np = row_keys(rp, pred.L), no = row_keys(ro, pred.L);
    unsigned long long inter = 0;
    for (int64_t t = lane; t < static_cast<int64_t>(rp.count) * rp.expand; t += 32) {
        const int64_t j = key_at(rp, t);
        if (j < pred.L && contains(ro, j)) ++inter;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) inter += __shfl_xor_sync(0xffffffffu, inter, o);
    if (lane == 0) {
        atomicAdd(out, inter);
        atomicAdd(out + 1, static_cast<unsigned long long>(np));
        if (np != no) atomicAdd(out + 2, 1ull);
    }
}

}  // namespace

void run_prediction_accuracy(const AttnArgs& pred, const AttnArgs& orc, unsigned long long* out, cudaStream_t st) {
    const unsigned grid = static_cast<unsigned>(ceil_div_i(pred.pairs * pred.L, kWarps));
    accuracy_kernel<<<grid, kWarps * 32, 0, st>>>(pred, orc, out);
    note_launch();
}

}  // namespace dsa
