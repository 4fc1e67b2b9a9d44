// Mask accounting on the device: prediction_accuracy
// (P/src/maskgen.cpp:94-107) between two masks of one layout --
// |pred n oracle| / |pred|, per-row counts required equal -- and the
// reference's dataflow fetch-count model (P/src/dataflow.cpp:10-62), the
// cost model SURVEY 8(f)4 names for grouping query rows.
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

// The reference's dataflow::simulate (P/src/dataflow.cpp:10-62) for one
// band of `band` consecutive rows (band <= 32: lane r = row first + r), one
// warp per (pair, band):
//   idle       = sum over rows of (band max kept - own kept)   (:13-18)
//   kind 0  row_by_row               fetches = nnz (band 1)     (:21-24)
//   kind 1  row_parallel             step t: one fetch per distinct t-th
//                                    kept column of the band    (:25-33)
//   kind 2  row_parallel_reordered   |union of the band's rows| (:34-40)
// (kind 2: a per-warp bit set over the L keys in shared memory)
constexpr int kDfWarps = 4;
__global__ void __launch_bounds__(kDfWarps * 32) dataflow_kernel(AttnArgs m, int band, int kind,
                                                                 unsigned long long* __restrict__ fetches,
                                                                 unsigned long long* __restrict__ idle) {
    extern __shared__ uint32_t bits_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nbands = (m.L + band - 1) / band;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * kDfWarps + warp;
    const bool live_w = w < m.pairs * nbands;
    const int64_t pair = live_w ? w / nbands : 0;
    const int64_t first = live_w ? (w % nbands) * band : 0;
    const int rows = live_w ? static_cast<int>(m.L - first < band ? m.L - first : band) : 0;
    const bool mine = lane < rows;
    RowList rl{nullptr, 0, 1};
    int64_t n = 0;
    if (mine) {
        rl = row_list(m, pair, first + lane);
        n = row_keys(rl, m.L);
    }
    int64_t mx = n;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    unsigned long long idl = mine ? static_cast<unsigned long long>(mx - n) : 0ull, f = 0;
    if (kind == 0) {
        f = static_cast<unsigned long long>(n);
        idl = 0;
    } else if (kind == 1) {
        for (int64_t t = 0; t < mx; ++t) {
            const bool act = mine && t < n;
            const unsigned am = __ballot_sync(0xffffffffu, act);
            const uint32_t key = act ? static_cast<uint32_t>(key_at(rl, t)) : 0xffffffffu;
            const unsigned same = __match_any_sync(0xffffffffu, key);
            // one fetch per distinct key among the active lanes: its lowest lane
            if (act && (__ffs(same & am) - 1) == lane) ++f;
        }
    } else {
        uint32_t* bits = bits_all + warp * ((m.L + 31) / 32);
        const int64_t nw = (m.L + 31) / 32;
        for (int64_t i = lane; i < nw; i += 32) bits[i] = 0u;
        __syncwarp();
        if (mine)
            for (int64_t t = 0; t < n; ++t) {
                const int64_t j = key_at(rl, t);
                atomicOr(&bits[j >> 5], 1u << (j & 31));
            }
        __syncwarp();
        for (int64_t i = lane; i < nw; i += 32) f += static_cast<unsigned long long>(__popc(bits[i]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        f += __shfl_xor_sync(0xffffffffu, f, o);
        idl += __shfl_xor_sync(0xffffffffu, idl, o);
    }
    if (lane == 0 && live_w) {
        atomicAdd(fetches + pair, f);
        atomicAdd(idle + pair, idl);
    }
}

}  // namespace

void run_dataflow(const AttnArgs& m, int band, int kind, unsigned long long* fetches, unsigned long long* idle,
                  cudaStream_t st) {
    const int64_t nbands = ceil_div_i(m.L, band);
    const unsigned grid = static_cast<unsigned>(ceil_div_i(m.pairs * nbands, kDfWarps));
    const size_t smem = kind == 2 ? static_cast<size_t>(kDfWarps) * ceil_div_i(m.L, 32) * 4 : 0;
    if (smem > 48 * 1024) cudaFuncSetAttribute(dataflow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    dataflow_kernel<<<grid, kDfWarps * 32, smem, st>>>(m, band, kind, fetches, idle);
    note_launch();
}

void run_prediction_accuracy(const AttnArgs& pred, const AttnArgs& orc, unsigned long long* out, cudaStream_t st) {
    const unsigned grid = static_cast<unsigned>(ceil_div_i(pred.pairs * pred.L, kWarps));
    accuracy_kernel<<<grid, kWarps * 32, 0, st>>>(pred, orc, out);
    note_launch();
}

}  // namespace dsa
