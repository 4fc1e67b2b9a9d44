// C-ABI entry points (include/dsa_b200.h): validation, workspace planning
// and stream-ordered launches of the sm_100a kernels.  No exceptions cross
// this boundary; errors become dsa_status codes + dsa_last_error().
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "dsa_b200.h"
#include "dsa_internal.h"
#include "kernels.h"

#define DSA_STR2(x) #x
#define DSA_STR(x) DSA_STR2(x)

namespace dsa {

namespace {
thread_local std::string g_last_error;

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

int64_t pairs_of(const dsa_config& c) { return c.batch * c.heads; }
int qmax_of(int bits) { return (1 << (bits - 1)) - 1; }
int64_t span_of(const dsa_config& c) {
    const int64_t q = qmax_of(c.bits);
    return 2 * c.k * q * q + 1;
}
int64_t nbands(const dsa_config& c) {
    return c.mask_mode == DSA_MASK_COLVEC ? ceil_div(c.L, c.vec_v)
           : c.mask_mode == DSA_MASK_BLOCK ? ceil_div(c.L, c.block)
                                           : c.L;
}

void check_cuda(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw_cuda(e, where);
}

void validate(const dsa_config* cp) {
    if (!cp) throw Error(DSA_ERR_PARAM, "dsa: null config");
    const dsa_config& c = *cp;
    if (c.batch < 1 || c.heads < 1) throw Error(DSA_ERR_SHAPE, "dsa: batch and heads must be >= 1");
    // pairs index grid.y / grid.z of the launches (<= 65535, and 2 x pairs for
    // the quantise pass) and 24 bits of the deferred-level list entries
    if (c.batch * c.heads >= 32768)
        throw Error(DSA_ERR_SHAPE, "dsa: batch * heads must be < 32768 per call (split the batch)");
    if (c.L < 1) throw Error(DSA_ERR_SHAPE, "Matrix: dimensions must be positive");
    if (c.L >= (int64_t{1} << 31)) throw Error(DSA_ERR_SHAPE, "dsa: L must be < 2^31");
    if (c.d != 16 && c.d != 32 && c.d != 64 && c.d != 128)
        throw Error(DSA_ERR_UNSUPPORTED, "dsa: head dim d must be one of 16, 32, 64, 128");
    if (c.k != 16 && c.k != 32) throw Error(DSA_ERR_UNSUPPORTED, "dsa: projection width k must be 16 or 32");
    if (c.k > c.d) throw Error(DSA_ERR_PARAM, "init_projection: need 1 <= k <= d");
    if (c.dtype != DSA_F32 && c.dtype != DSA_BF16) throw Error(DSA_ERR_PARAM, "dsa: dtype must be F32 or BF16");
    if (c.bits != 2 && c.bits != 4 && c.bits != 8) {
        if (c.bits == 0 || c.bits == 16)
            throw Error(DSA_ERR_UNSUPPORTED, "dsa: full/16-bit prediction levels are not integer-exact on the tensor-core path");
        throw Error(DSA_ERR_PARAM, "QuantSpec: bits must be one of {2,4,8,16,full}");
    }
    if (c.quant_scope != DSA_QUANT_PER_TENSOR && c.quant_scope != DSA_QUANT_PER_ROW)
        throw Error(DSA_ERR_PARAM, "dsa: unknown quant_scope");
    switch (c.mask_mode) {
        case DSA_MASK_ROW_TOPK:
            if (c.keep < 1 || c.keep > c.L) throw Error(DSA_ERR_PARAM, "row_topk_indices: k_keep out of range");
            if (c.L * (c.quant_scope == DSA_QUANT_PER_ROW ? 8 : 4) > 200 * 1024)
                throw Error(DSA_ERR_UNSUPPORTED, "dsa: row top-k supports L <= 51200 (25600 per-row)");
            break;
        case DSA_MASK_COLVEC:
            if (c.vec_v < 1) throw Error(DSA_ERR_PARAM, "colvec_mask: vector height must be >= 1");
            if (c.keep < 1 || c.keep > c.L) throw Error(DSA_ERR_PARAM, "row_topk_indices: k_keep out of range");
            if (c.quant_scope != DSA_QUANT_PER_TENSOR)
                throw Error(DSA_ERR_UNSUPPORTED, "dsa: colvec mode needs per-tensor levels");
            if (c.L * 4 > 200 * 1024) throw Error(DSA_ERR_UNSUPPORTED, "dsa: colvec supports L <= 51200");
            break;
        case DSA_MASK_BLOCK:
            if (c.block < 1) throw Error(DSA_ERR_PARAM, "dsa: block must be >= 1");
            if (c.keep < 1 || c.keep > ceil_div(c.L, c.block))
                throw Error(DSA_ERR_PARAM, "row_topk_indices: k_keep out of range");
            if (c.quant_scope != DSA_QUANT_PER_TENSOR)
                throw Error(DSA_ERR_UNSUPPORTED, "dsa: block mode needs per-tensor levels");
            break;
        case DSA_MASK_THRESHOLD:
            if (c.frac_num < 1 || c.frac_den < 1) throw Error(DSA_ERR_PARAM, "threshold_mask: theta must be finite");
            if (c.cap < 1) throw Error(DSA_ERR_PARAM, "dsa: cap must be >= 1");
            if (c.quant_scope != DSA_QUANT_PER_TENSOR)
                throw Error(DSA_ERR_UNSUPPORTED, "dsa: threshold mode needs per-tensor levels");
            if (c.L * 4 > 200 * 1024) throw Error(DSA_ERR_UNSUPPORTED, "dsa: threshold supports L <= 51200");
            if (c.frac_num * c.L > (int64_t{1} << 22)) throw Error(DSA_ERR_PARAM, "dsa: frac_num * L too large");
            break;
        default: throw Error(DSA_ERR_PARAM, "dsa: unknown mask_mode");
    }
}

int64_t capacity_of(const dsa_config& c) {
    const int64_t P = pairs_of(c);
    switch (c.mask_mode) {
        case DSA_MASK_ROW_TOPK: return P * c.L * c.keep;
        case DSA_MASK_COLVEC: return P * ceil_div(c.L, c.vec_v) * c.keep;
        case DSA_MASK_BLOCK: return P * ceil_div(c.L, c.block) * c.keep;
        default: {
            // sum_i <= 1 => at most floor(L * num / den) keys reach theta.
            const int64_t bound = std::min<int64_t>(c.cap, (c.L * c.frac_num) / c.frac_den);
            int64_t per_pair = 0;
            if (c.causal) {
                // rows i < bound keep at most i + 1 candidates, the rest `bound`
                const int64_t b = std::min<int64_t>(std::max<int64_t>(bound, 0), c.L);
                per_pair = (b * (b + 1)) / 2 + (c.L - b) * b;
            } else {
                per_pair = c.L * bound;
            }
            return P * std::max<int64_t>(per_pair, 1);
        }
    }
}

constexpr int kMaxChunks = 4;  // dsa_pipeline: pair chunks overlapped on three streams

// Workspace: [x64 | amax | pimg | pooled | etab | counts | cut | scan | levels | scales | mask]
struct Plan {
    size_t x64 = 0, xhat = 0, amax = 0, pimg = 0, ovf = 0, pooled = 0, etab = 0, counts = 0, cut = 0, scan = 0, lq = 0, lk = 0, sq = 0,
           sk = 0, cols = 0, rowptr = 0, total = 0;
    size_t scan_bytes = 0;
    bool has_xhat = false;
};

Plan plan(const dsa_config& c, bool pipeline, bool own_mask) {
    Plan p;
    const int64_t P = pairs_of(c);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += align_up(bytes);
        return o;
    };
    const bool per_tensor = c.quant_scope == DSA_QUANT_PER_TENSOR;
    // the f64 projection scratch only serves the fallback kernels (f32 inputs,
    // other d, or DSA_PREDICT_DFMA); the tensor-core path needs the P image
    const bool tc_path = c.dtype == DSA_BF16 && (c.d == 64 || c.d == 128) && (c.k == 16 || c.k == 32);
    const bool need_x64 = per_tensor && (!tc_path || options().predict_dfma);
    p.x64 = take(need_x64 ? sizeof(double) * P * 2 * c.L * c.k : 0);
    // stored x^ for the streaming quantise pass.  Uncertified
    // levels go to a deferred list (quantize_fix_kernel).  8-bit configs keep
    // the two-read pass: with x^ they measured slower (C3 0.533 vs 0.471 ms:
    // the amax pass of the d = 128 shape is latency-bound and the x^ writes
    // lengthen it).
    // (the tile kernels only run for L > 16384 or under DSA_PREDICT_TILES:
    // the per-tensor CTA kernels of project_tensor.cu take the rest)
    p.has_xhat = per_tensor && tc_path && c.bits <= 4 && !options().predict_dfma &&
                 (options().predict_tiles || c.L > 128 * 128);
    p.xhat = take(p.has_xhat ? sizeof(float) * P * xhat_floats_per_pair(c.L, c.k) : 0);
    p.amax = take(per_tensor ? sizeof(unsigned long long) * P * 2 : 0);
    p.pimg = take(tc_path ? align_up(predict_tc_image_bytes(c.d, c.k)) * kMaxChunks : 0);
    const bool row_scaled = c.mask_mode == DSA_MASK_ROW_TOPK && !per_tensor;
    p.ovf = take(row_scaled ? 16 + sizeof(int64_t) * P * c.L : 0);  // overflow count + row list
    p.pooled = take(c.mask_mode == DSA_MASK_BLOCK ? sizeof(int32_t) * P * 2 * ceil_div(c.L, c.block) * c.k : 0);
    p.etab = take(c.mask_mode == DSA_MASK_THRESHOLD ? sizeof(int64_t) * P * span_of(c) : 0);
    p.counts = take(c.mask_mode == DSA_MASK_THRESHOLD ? sizeof(uint64_t) * P * c.L : 0);
    p.cut = take(c.mask_mode == DSA_MASK_THRESHOLD ? sizeof(int2) * P * c.L : 0);
    if (c.mask_mode == DSA_MASK_THRESHOLD) p.scan_bytes = select_scan_tmp_bytes(P * c.L);
    p.scan = take(p.scan_bytes);
    if (pipeline) {
        p.lq = take(sizeof(uint16_t) * P * c.L * c.k);
        p.lk = take(sizeof(uint16_t) * P * c.L * c.k);
        const int64_t ns = per_tensor ? P : P * c.L;
        p.sq = take(sizeof(double) * ns);
        p.sk = take(sizeof(double) * ns);
        if (own_mask) {
            p.cols = take(sizeof(uint32_t) * capacity_of(c));
            p.rowptr = take(c.mask_mode == DSA_MASK_THRESHOLD ? sizeof(uint64_t) * (P * c.L + 1) : 0);
        }
    }
    p.total = off;
    return p;
}

template <class T>
T* at(void* ws, size_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

void check_ws(const Plan& p, void* ws, size_t bytes) {
    if (p.total > 0 && (!ws || bytes < p.total))
        throw Error(DSA_ERR_PARAM, "dsa: workspace too small (need " + std::to_string(p.total) + " bytes)");
}

// Phase scratch of the pairs [pair0, ...) of the planned config `c`; chunk
// `ci` gets its own P-split image (concurrent chunks never share scratch).
struct Scratch {
    double* x64;
    float* xhat;
    unsigned long long* amax;
    unsigned char* pimg;
    int32_t* pooled;
    int64_t* etab;
    uint64_t* counts;
    int2* cut;
    void* scan;
    size_t scan_bytes;
    unsigned* ovf_n;
    int64_t* ovf_list;
};

Scratch scratch_of(const dsa_config& c, const Plan& pl, void* ws, int64_t pair0 = 0, int ci = 0) {
    Scratch r{};
    r.x64 = at<double>(ws, pl.x64) + pair0 * 2 * c.L * c.k;
    r.xhat = pl.has_xhat ? at<float>(ws, pl.xhat) + pair0 * xhat_floats_per_pair(c.L, c.k) : nullptr;
    r.amax = at<unsigned long long>(ws, pl.amax) + pair0 * 2;
    const bool tc_path = c.dtype == DSA_BF16 && (c.d == 64 || c.d == 128) && (c.k == 16 || c.k == 32);
    r.pimg = tc_path ? at<unsigned char>(ws, pl.pimg) + static_cast<size_t>(ci) * align_up(predict_tc_image_bytes(c.d, c.k))
                     : nullptr;
    r.pooled = at<int32_t>(ws, pl.pooled) + pair0 * 2 * ceil_div(c.L, c.block > 0 ? c.block : 1) * c.k;
    r.etab = at<int64_t>(ws, pl.etab);
    r.counts = at<uint64_t>(ws, pl.counts);
    r.cut = c.mask_mode == DSA_MASK_THRESHOLD ? at<int2>(ws, pl.cut) : nullptr;
    r.scan = at<void>(ws, pl.scan);
    r.scan_bytes = pl.scan_bytes;
    const bool row_scaled = c.mask_mode == DSA_MASK_ROW_TOPK && c.quant_scope != DSA_QUANT_PER_TENSOR;
    r.ovf_n = row_scaled ? at<unsigned>(ws, pl.ovf) + pair0 * 0 : nullptr;
    r.ovf_list = row_scaled ? reinterpret_cast<int64_t*>(at<char>(ws, pl.ovf) + 16) : nullptr;
    return r;
}

// Number of pair chunks dsa_pipeline overlaps (1 = serial).  Threshold
// masks keep one global CSR (a single scan over all rows): serial.
int pipeline_chunks(const dsa_config& c) {
    const int env = options().pipeline_chunks;
    if (c.mask_mode == DSA_MASK_THRESHOLD) return 1;
    const int64_t P = pairs_of(c);
    // default serial: measured on B200 (C2), 2 and 4 chunks on three streams
    // were 1-2 % slower than back-to-back full-width kernels
    int n = env >= 1 ? env : 1;
    n = static_cast<int>(std::min<int64_t>(std::min(n, kMaxChunks), P / 2));
    return n < 2 ? 1 : n;
}

struct StreamSet {
    cudaStream_t s[3];
    cudaEvent_t fork, join, ev[2 * kMaxChunks];
};

// Per-device streams/events for dsa_pipeline (created once, never freed).
StreamSet& stream_set() {
    static std::mutex mu;
    static std::vector<StreamSet*> sets;
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(mu);
    if (static_cast<int>(sets.size()) <= dev) sets.resize(dev + 1, nullptr);
    if (!sets[dev]) {
        auto* x = new StreamSet;
        for (auto& st : x->s) check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        check_cuda(cudaEventCreateWithFlags(&x->fork, cudaEventDisableTiming), "event");
        check_cuda(cudaEventCreateWithFlags(&x->join, cudaEventDisableTiming), "event");
        for (auto& e : x->ev) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        sets[dev] = x;
    }
    return *sets[dev];
}

void do_predict(const dsa_config& c, const void* q, const void* k, const float* p, uint16_t* lq,
                uint16_t* lk, double* sq, double* sk, const Scratch& ws, cudaStream_t st) {
    if (!q || !k || !p || !lq || !lk || !sq || !sk) throw Error(DSA_ERR_PARAM, "dsa_predict: null pointer");
    PredictArgs a{};
    a.q = q;
    a.k = k;
    a.p = p;
    a.pairs = pairs_of(c);
    a.L = c.L;
    a.D = c.d;
    a.KD = c.k;
    a.bf16 = c.dtype == DSA_BF16;
    a.per_row = c.quant_scope == DSA_QUANT_PER_ROW;
    a.round_f32 = c.round_proj_f32;
    a.qmax = static_cast<double>(qmax_of(c.bits));
    a.lq = lq;
    a.lk = lk;
    a.sq = sq;
    a.sk = sk;
    a.xws = ws.x64;
    a.xhat = ws.xhat;
    a.amax = ws.amax;
    a.pimg = ws.pimg;
    run_predict(a, st);
    check_cuda(cudaGetLastError(), "dsa_predict launch");
}

SelectArgs select_args(const dsa_config& c, const uint16_t* lq, const uint16_t* lk, const double* sq,
                       const double* sk, const dsa_mask& m, const Scratch& ws) {
    SelectArgs a{};
    a.mode = c.mask_mode;
    a.pairs = pairs_of(c);
    a.L = c.L;
    a.KD = c.k;
    a.D = c.d;
    a.per_row = c.quant_scope == DSA_QUANT_PER_ROW;
    a.lq = lq;
    a.lk = lk;
    a.sq = sq;
    a.sk = sk;
    a.keep = c.keep;
    a.vec_v = c.vec_v;
    a.block = c.block;
    a.force_diag = c.force_diag;
    a.causal = c.causal;
    a.frac_num = c.frac_num;
    a.frac_den = c.frac_den;
    a.cap = c.cap;
    a.qmax = qmax_of(c.bits);
    a.cols = m.cols;
    a.rowptr = m.rowptr;
    a.capacity = m.capacity;
    a.empty_rows = m.empty_rows;
    a.pooled = ws.pooled;
    a.etab = ws.etab;
    a.counts = ws.counts;
    a.cut = ws.cut;
    a.span = span_of(c);
    a.scan_tmp = ws.scan;
    a.scan_tmp_bytes = ws.scan_bytes;
    a.ovf_n = ws.ovf_n;
    a.ovf_list = ws.ovf_list;
    return a;
}

void do_select(const dsa_config& c, const uint16_t* lq, const uint16_t* lk, const double* sq,
               const double* sk, const dsa_mask& m, const Scratch& ws, cudaStream_t st) {
    if (!lq || !lk || !sq || !sk || !m.cols) throw Error(DSA_ERR_PARAM, "dsa_select: null pointer");
    if (m.capacity < capacity_of(c) && c.mask_mode != DSA_MASK_THRESHOLD)
        throw Error(DSA_ERR_PARAM, "dsa_select: mask capacity too small");
    if (c.mask_mode == DSA_MASK_THRESHOLD && (!m.rowptr || m.capacity < capacity_of(c)))
        throw Error(DSA_ERR_PARAM, "dsa_select: threshold mode needs rowptr and capacity >= dsa_mask_capacity()");
    const SelectArgs a = select_args(c, lq, lk, sq, sk, m, ws);
    if (m.empty_rows && c.mask_mode != DSA_MASK_THRESHOLD)
        check_cuda(cudaMemsetAsync(m.empty_rows, 0, pairs_of(c) * c.L, st), "dsa_select memset");
    run_select(a, st);
    check_cuda(cudaGetLastError(), "dsa_select launch");
}

AttnArgs attn_args(const dsa_config& c, const void* q, const void* k, const void* v, const dsa_mask& m, void* z) {
    AttnArgs a{};
    a.mode = c.mask_mode;
    a.pairs = pairs_of(c);
    a.L = c.L;
    a.D = c.d;
    a.bf16 = c.dtype == DSA_BF16;
    a.scale = c.scale;
    a.q = q;
    a.k = k;
    a.v = v;
    a.cols = m.cols;
    a.rowptr = m.rowptr;
    a.keep = c.keep;
    a.vec_v = c.vec_v;
    a.block = c.block;
    a.z = z;
    a.empty_rows = m.empty_rows;
    return a;
}

void do_attention(const dsa_config& c, const void* q, const void* k, const void* v,
                  const dsa_mask& m, void* z, cudaStream_t st) {
    if (!q || !k || !v || !z || !m.cols) throw Error(DSA_ERR_PARAM, "dsa_sparse_attention: null pointer");
    if (c.mask_mode == DSA_MASK_THRESHOLD && !m.rowptr)
        throw Error(DSA_ERR_PARAM, "dsa_sparse_attention: threshold mask needs rowptr");
    run_attention(attn_args(c, q, k, v, m, z), st);
    check_cuda(cudaGetLastError(), "dsa_sparse_attention launch");
}

// COLVEC select + attention in one kernel when supported; with no caller
// mask the selected lists stay on chip (nothing written to HBM).
bool try_fused(const dsa_config& c, const void* q, const void* k, const void* v, const uint16_t* lq,
               const uint16_t* lk, const double* sq, const double* sk, const dsa_mask& m, bool mask_wanted,
               void* z, const Scratch& ws, cudaStream_t st) {
    if (c.mask_mode != DSA_MASK_COLVEC) return false;
    SelectArgs sa = select_args(c, lq, lk, sq, sk, m, ws);
    const AttnArgs aa = attn_args(c, q, k, v, m, z);
    if (!colvec_fused_supported(sa, aa)) return false;
    if (!mask_wanted) sa.cols = nullptr;
    if (m.empty_rows) check_cuda(cudaMemsetAsync(m.empty_rows, 0, pairs_of(c) * c.L, st), "dsa_pipeline memset");
    run_colvec_fused(sa, aa, st);
    check_cuda(cudaGetLastError(), "dsa_pipeline fused launch");
    return true;
}

void require_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw Error(DSA_ERR_CUDA, "dsa: no CUDA device available (the B200 path has no CPU fallback)");
}

}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }

static std::atomic<uint64_t> g_launches{0};

namespace {
bool env_flag(const char* name) {
    const char* e = std::getenv(name);
    return e != nullptr && *e != '\0' && std::strcmp(e, "0") != 0;
}
Options read_options() {
    Options o{};
    o.attn_generic = env_flag("DSA_ATTN_GENERIC");
    o.threshold_generic = env_flag("DSA_THRESHOLD_GENERIC");
    o.block_generic = env_flag("DSA_BLOCK_GENERIC");
    o.topk_generic = env_flag("DSA_TOPK_GENERIC");
    o.predict_dfma = env_flag("DSA_PREDICT_DFMA");
    o.fuse = env_flag("DSA_FUSE");
    o.block_tc = env_flag("DSA_BLOCK_TC");
    o.predict_tiles = env_flag("DSA_PREDICT_TILES");
    o.block_cpasync = env_flag("DSA_BLOCK_CPASYNC");
    const char* e = std::getenv("DSA_PIPELINE_CHUNKS");
    o.pipeline_chunks = e ? std::atoi(e) : -1;
    return o;
}
// read once, when the shared library is loaded
const Options g_options = read_options();
}  // namespace

const Options& options() { return g_options; }

int sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    int n = cache[dev].load(std::memory_order_relaxed);
    if (n == 0) {
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}
void note_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n), std::memory_order_relaxed); }

[[noreturn]] void throw_unsupported(const std::string& what) { throw Error(DSA_ERR_UNSUPPORTED, "dsa: " + what); }
[[noreturn]] void throw_cuda(cudaError_t e, const char* where) {
    throw Error(DSA_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

}  // namespace dsa

using namespace dsa;

extern "C" {

int dsa_abi_version(void) { return DSA_ABI_VERSION; }
uint64_t dsa_launch_counter(void) { return g_launches.load(std::memory_order_relaxed); }
const char* dsa_last_error(void) { return g_last_error.c_str(); }
const char* dsa_build_info(void) {
    return "dsa_b200 sm_100a, CUDA runtime " DSA_STR(CUDART_VERSION);
}

dsa_status dsa_config_validate(const dsa_config* cfg) {
    return guard([&] { validate(cfg); });
}

size_t dsa_workspace_bytes(const dsa_config* cfg) {
    size_t out = 0;
    dsa_status s = guard([&] {
        validate(cfg);
        out = plan(*cfg, true, true).total;
    });
    return s == DSA_OK ? out : 0;
}

int64_t dsa_mask_capacity(const dsa_config* cfg) {
    int64_t out = -1;
    guard([&] {
        validate(cfg);
        out = capacity_of(*cfg);
    });
    return out;
}

dsa_status dsa_predict(const dsa_config* cfg, const void* q, const void* k, const float* p,
                       uint16_t* levels_q, uint16_t* levels_k, double* scale_q, double* scale_k,
                       void* workspace, size_t workspace_bytes, void* stream) {
    return guard([&] {
        validate(cfg);
        require_device();
        Plan pl = plan(*cfg, false, false);
        check_ws(pl, workspace, workspace_bytes);
        do_predict(*cfg, q, k, p, levels_q, levels_k, scale_q, scale_k, scratch_of(*cfg, pl, workspace),
                   static_cast<cudaStream_t>(stream));
    });
}

size_t dsa_predict_wtilde_workspace_bytes(const dsa_config* cfg) {
    size_t out = 0;
    dsa_status s = guard([&] {
        validate(cfg);
        const int64_t P = pairs_of(*cfg);
        out = cfg->quant_scope == DSA_QUANT_PER_TENSOR
                  ? align_up(sizeof(double) * P * 2 * cfg->L * cfg->k) + align_up(sizeof(unsigned long long) * P * 2)
                  : 0;
    });
    return s == DSA_OK ? out : 0;
}

dsa_status dsa_predict_wtilde(const dsa_config* cfg, int64_t d_model, const double* x, const double* p,
                              double* r, const double* wq, const double* wk, uint16_t* levels_q,
                              uint16_t* levels_k, double* scale_q, double* scale_k, void* workspace,
                              size_t workspace_bytes, void* stream) {
    return guard([&] {
        validate(cfg);
        require_device();
        const dsa_config& c = *cfg;
        if (x && (d_model < 1 || !p)) throw Error(DSA_ERR_SHAPE, "approx_scores: X feature dim != d");
        if (!r || !wq || !wk || !levels_q || !levels_k || !scale_q || !scale_k)
            throw Error(DSA_ERR_PARAM, "dsa_predict_wtilde: null pointer");
        const size_t need = dsa_predict_wtilde_workspace_bytes(cfg);
        if (need > 0 && (!workspace || workspace_bytes < need))
            throw Error(DSA_ERR_PARAM, "dsa: workspace too small (need " + std::to_string(need) + " bytes)");
        WtildeArgs a{};
        a.batch = c.batch;
        a.heads = c.heads;
        a.L = c.L;
        a.dm = d_model;
        a.KD = c.k;
        a.x = x;
        a.p = p;
        a.r = r;
        a.wq = wq;
        a.wk = wk;
        a.round_f32 = c.round_proj_f32;
        a.per_row = c.quant_scope == DSA_QUANT_PER_ROW;
        a.qmax = static_cast<double>(qmax_of(c.bits));
        a.lq = levels_q;
        a.lk = levels_k;
        a.sq = scale_q;
        a.sk = scale_k;
        if (!a.per_row) {
            a.x64 = static_cast<double*>(workspace);
            a.amax = reinterpret_cast<unsigned long long*>(static_cast<char*>(workspace) +
                                                           align_up(sizeof(double) * pairs_of(c) * 2 * c.L * c.k));
        }
        run_predict_wtilde(a, static_cast<cudaStream_t>(stream));
        check_cuda(cudaGetLastError(), "dsa_predict_wtilde launch");
    });
}

dsa_status dsa_select(const dsa_config* cfg, const uint16_t* levels_q, const uint16_t* levels_k,
                      const double* scale_q, const double* scale_k, const dsa_mask* mask,
                      void* workspace, size_t workspace_bytes, void* stream) {
    return guard([&] {
        validate(cfg);
        require_device();
        if (!mask) throw Error(DSA_ERR_PARAM, "dsa_select: null mask");
        Plan pl = plan(*cfg, false, false);
        check_ws(pl, workspace, workspace_bytes);
        do_select(*cfg, levels_q, levels_k, scale_q, scale_k, *mask, scratch_of(*cfg, pl, workspace),
                  static_cast<cudaStream_t>(stream));
    });
}

dsa_status dsa_project_qkv(int64_t batch, int64_t L, int64_t d_model, int64_t heads, int64_t dk,
                           int64_t dv, int64_t npred, const void* x, const void* w, void* q,
                           void* k, void* v, float* r, void* stream) {
    return guard([&] {
        if (batch < 1 || L < 1 || heads < 1 || d_model < 1 || dk < 1 || dv < 1)
            throw Error(DSA_ERR_SHAPE, "dsa_project_qkv: sizes must be >= 1");
        if (d_model % 64 != 0) throw Error(DSA_ERR_UNSUPPORTED, "dsa_project_qkv: d_model must be a multiple of 64");
        if (dk % 32 != 0 || dv % 32 != 0)
            throw Error(DSA_ERR_UNSUPPORTED, "dsa_project_qkv: d_k and d_v must be multiples of 32");
        if (npred < 0 || npred > 32) throw Error(DSA_ERR_PARAM, "dsa_project_qkv: npred must be in [0, 32]");
        if (!x || !w || !q || !k || !v || (npred > 0 && !r))
            throw Error(DSA_ERR_PARAM, "dsa_project_qkv: null pointer");
        if (batch * L >= (int64_t{1} << 31) || heads * (2 * dk + dv) + npred >= (int64_t{1} << 31))
            throw Error(DSA_ERR_SHAPE, "dsa_project_qkv: operand too large for 32-bit TMA coordinates");
        require_device();
        QkvGemmArgs g{batch, L, d_model, heads, dk, dv, npred, x, w, q, k, v, r};
        run_qkv_gemm(g, static_cast<cudaStream_t>(stream));
        check_cuda(cudaGetLastError(), "dsa_project_qkv launch");
    });
}

dsa_status dsa_sparse_attention(const dsa_config* cfg, const void* q, const void* k,
                                const void* v, const dsa_mask* mask, void* z, void* stream) {
    return guard([&] {
        validate(cfg);
        require_device();
        if (!mask) throw Error(DSA_ERR_PARAM, "dsa_sparse_attention: null mask");
        do_attention(*cfg, q, k, v, *mask, z, static_cast<cudaStream_t>(stream));
    });
}

dsa_status dsa_pipeline(const dsa_config* cfg, const void* q, const void* k, const void* v,
                        const float* p, void* z, const dsa_mask* mask_out, void* workspace,
                        size_t workspace_bytes, void* stream) {
    return guard([&] {
        validate(cfg);
        require_device();
        const dsa_config& c = *cfg;
        Plan pl = plan(c, true, mask_out == nullptr);
        check_ws(pl, workspace, workspace_bytes);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        uint16_t* lq = at<uint16_t>(workspace, pl.lq);
        uint16_t* lk = at<uint16_t>(workspace, pl.lk);
        double* sq = at<double>(workspace, pl.sq);
        double* sk = at<double>(workspace, pl.sk);
        dsa_mask m{};
        if (mask_out) {
            m = *mask_out;
        } else {
            m.cols = at<uint32_t>(workspace, pl.cols);
            m.rowptr = c.mask_mode == DSA_MASK_THRESHOLD ? at<uint64_t>(workspace, pl.rowptr) : nullptr;
            m.capacity = capacity_of(c);
            m.empty_rows = nullptr;
        }
        const int64_t P = pairs_of(c);
        const int nch = pipeline_chunks(c);
        if (nch <= 1) {
            const Scratch sc = scratch_of(c, pl, workspace);
            do_predict(c, q, k, p, lq, lk, sq, sk, sc, st);
            if (try_fused(c, q, k, v, lq, lk, sq, sk, m, mask_out != nullptr, z, sc, st)) return;
            do_select(c, lq, lk, sq, sk, m, sc, st);
            do_attention(c, q, k, v, m, z, st);
            return;
        }
        // pair chunks: predict(c+1) || select(c) || attention(c-1) on three
        // streams (event fork/join off the caller's stream; graph-capturable)
        StreamSet& ss = stream_set();
        check_cuda(cudaEventRecord(ss.fork, st), "dsa_pipeline fork");
        for (int i = 0; i < 3; ++i) check_cuda(cudaStreamWaitEvent(ss.s[i], ss.fork, 0), "dsa_pipeline fork");
        const size_t esz = c.dtype == DSA_BF16 ? 2 : 4;
        const int64_t per_scale = c.quant_scope == DSA_QUANT_PER_TENSOR ? 1 : c.L;
        const int64_t per_cols = capacity_of(c) / P;
        for (int ci = 0; ci < nch; ++ci) {
            const int64_t p0 = P * ci / nch, p1 = P * (ci + 1) / nch;
            dsa_config cc = c;
            cc.batch = p1 - p0;
            cc.heads = 1;
            const Scratch sc = scratch_of(c, pl, workspace, p0, ci);
            const size_t xo = static_cast<size_t>(p0 * c.L * c.d) * esz;
            const auto* qc = static_cast<const char*>(q) + xo;
            const auto* kc = static_cast<const char*>(k) + xo;
            const auto* vc = static_cast<const char*>(v) + xo;
            auto* zc = static_cast<char*>(z) + xo;
            uint16_t* lqc = lq + p0 * c.L * c.k;
            uint16_t* lkc = lk + p0 * c.L * c.k;
            double* sqc = sq + p0 * per_scale;
            double* skc = sk + p0 * per_scale;
            dsa_mask mc = m;
            mc.cols = m.cols + p0 * per_cols;
            mc.capacity = (p1 - p0) * per_cols;
            mc.empty_rows = m.empty_rows ? m.empty_rows + p0 * c.L : nullptr;
            do_predict(cc, qc, kc, p, lqc, lkc, sqc, skc, sc, ss.s[0]);
            check_cuda(cudaEventRecord(ss.ev[2 * ci], ss.s[0]), "dsa_pipeline event");
            check_cuda(cudaStreamWaitEvent(ss.s[1], ss.ev[2 * ci], 0), "dsa_pipeline event");
            do_select(cc, lqc, lkc, sqc, skc, mc, sc, ss.s[1]);
            check_cuda(cudaEventRecord(ss.ev[2 * ci + 1], ss.s[1]), "dsa_pipeline event");
            check_cuda(cudaStreamWaitEvent(ss.s[2], ss.ev[2 * ci + 1], 0), "dsa_pipeline event");
            do_attention(cc, qc, kc, vc, mc, zc, ss.s[2]);
        }
        check_cuda(cudaEventRecord(ss.join, ss.s[2]), "dsa_pipeline join");
        check_cuda(cudaStreamWaitEvent(st, ss.join, 0), "dsa_pipeline join");
    });
}

dsa_status dsa_prediction_accuracy(const dsa_config* cfg, const dsa_mask* pred, const dsa_mask* oracle,
                                   double* accuracy, void* stream) {
    return guard([&] {
        validate(cfg);
        require_device();
        if (!pred || !oracle || !accuracy || !pred->cols || !oracle->cols)
            throw Error(DSA_ERR_PARAM, "dsa_prediction_accuracy: null pointer");
        if (cfg->mask_mode == DSA_MASK_THRESHOLD && (!pred->rowptr || !oracle->rowptr))
            throw Error(DSA_ERR_PARAM, "dsa_prediction_accuracy: threshold masks need rowptr");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        unsigned long long* d = nullptr;
        check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&d), 3 * sizeof(unsigned long long), st), "alloc");
        check_cuda(cudaMemsetAsync(d, 0, 3 * sizeof(unsigned long long), st), "memset");
        run_prediction_accuracy(attn_args(*cfg, nullptr, nullptr, nullptr, *pred, nullptr),
                                attn_args(*cfg, nullptr, nullptr, nullptr, *oracle, nullptr), d, st);
        unsigned long long h[3] = {0, 0, 0};
        check_cuda(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st), "copy");
        check_cuda(cudaFreeAsync(d, st), "free");
        check_cuda(cudaStreamSynchronize(st), "sync");
        if (h[2] != 0) throw Error(DSA_ERR_PARAM, "prediction_accuracy: per-row counts differ");
        if (h[1] == 0) throw Error(DSA_ERR_PARAM, "prediction_accuracy: empty masks");
        *accuracy = static_cast<double>(h[0]) / static_cast<double>(h[1]);
    });
}

dsa_status dsa_dataflow_trace(const dsa_config* cfg, const dsa_mask* mask, int32_t schedule, int64_t band,
                              uint64_t* fetches, uint64_t* idle, void* stream) {
    return guard([&] {
        validate(cfg);
        require_device();
        if (!mask || !mask->cols || !fetches || !idle) throw Error(DSA_ERR_PARAM, "dsa_dataflow_trace: null pointer");
        if (cfg->mask_mode == DSA_MASK_THRESHOLD && !mask->rowptr)
            throw Error(DSA_ERR_PARAM, "dsa_dataflow_trace: threshold masks need rowptr");
        if (schedule < 0 || schedule > 2) throw Error(DSA_ERR_PARAM, "dsa_dataflow_trace: unknown schedule");
        // the reference: "simulate: band height must be >= 1" (P/src/dataflow.cpp:49)
        if (band < 1) throw Error(DSA_ERR_PARAM, "simulate: band height must be >= 1");
        if (band > 32) throw Error(DSA_ERR_UNSUPPORTED, "dsa_dataflow_trace: band <= 32 rows");
        if (cfg->L > 65536) throw Error(DSA_ERR_UNSUPPORTED, "dsa_dataflow_trace: L <= 65536");
        const int64_t P = pairs_of(*cfg);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        unsigned long long* d = nullptr;
        check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&d), 2 * P * sizeof(unsigned long long), st), "alloc");
        check_cuda(cudaMemsetAsync(d, 0, 2 * P * sizeof(unsigned long long), st), "memset");
        run_dataflow(attn_args(*cfg, nullptr, nullptr, nullptr, *mask, nullptr), static_cast<int>(band), schedule, d,
                     d + P, st);
        check_cuda(cudaMemcpyAsync(fetches, d, P * sizeof(uint64_t), cudaMemcpyDeviceToHost, st), "copy");
        check_cuda(cudaMemcpyAsync(idle, d + P, P * sizeof(uint64_t), cudaMemcpyDeviceToHost, st), "copy");
        check_cuda(cudaFreeAsync(d, st), "free");
        check_cuda(cudaStreamSynchronize(st), "sync");
    });
}

dsa_status dsa_row_topk_f64(int64_t rows, int64_t cols, const double* scores, int64_t keep, uint32_t* out,
                            void* stream) {
    return guard([&] {
        require_device();
        if (rows < 0 || cols < 1) throw Error(DSA_ERR_SHAPE, "Matrix: dimensions must be positive");
        if (keep < 1 || keep > cols) throw Error(DSA_ERR_PARAM, "row_topk_indices: k_keep out of range");
        if (cols * 8 > 200 * 1024) throw Error(DSA_ERR_UNSUPPORTED, "dsa_row_topk_f64: cols <= 25600");
        if (rows > 2147483647) throw Error(DSA_ERR_SHAPE, "dsa_row_topk_f64: rows < 2^31");
        if (rows == 0) return;
        if (!scores || !out) throw Error(DSA_ERR_PARAM, "dsa_row_topk_f64: null pointer");
        run_row_topk_f64(scores, rows, cols, keep, out, static_cast<cudaStream_t>(stream));
        check_cuda(cudaGetLastError(), "dsa_row_topk_f64");
    });
}

dsa_status dsa_colvec_mask_f64(int64_t l, int64_t v, int64_t keep, const double* scores, uint32_t* band_cols,
                               void* stream) {
    return guard([&] {
        require_device();
        if (v < 1) throw Error(DSA_ERR_PARAM, "colvec_mask: vector height must be >= 1");
        if (l < 1) throw Error(DSA_ERR_SHAPE, "Matrix: dimensions must be positive");
        if (keep < 1 || keep > l) throw Error(DSA_ERR_PARAM, "row_topk_indices: k_keep out of range");
        if (l * 8 > 200 * 1024) throw Error(DSA_ERR_UNSUPPORTED, "dsa_colvec_mask_f64: l <= 25600");
        if (!scores || !band_cols) throw Error(DSA_ERR_PARAM, "dsa_colvec_mask_f64: null pointer");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int64_t nb = (l + v - 1) / v;
        double* pooled = nullptr;
        check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&pooled), static_cast<size_t>(nb * l) * 8, st), "alloc");
        run_band_abs_sum_f64(scores, l, v, pooled, st);
        run_row_topk_f64(pooled, nb, l, keep, band_cols, st);
        check_cuda(cudaFreeAsync(pooled, st), "free");
        check_cuda(cudaGetLastError(), "dsa_colvec_mask_f64");
    });
}

dsa_status dsa_threshold_mask_f64(int64_t rows, int64_t cols, const double* scores, double theta,
                                  int32_t post_softmax, int32_t round_f32, uint8_t* keep, void* stream) {
    return guard([&] {
        require_device();
        if (!std::isfinite(theta)) throw Error(DSA_ERR_PARAM, "threshold_mask: theta must be finite");
        if (rows < 1 || cols < 1) throw Error(DSA_ERR_SHAPE, "Matrix: dimensions must be positive");
        if (!scores || !keep) throw Error(DSA_ERR_PARAM, "dsa_threshold_mask_f64: null pointer");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        double* scratch = nullptr;
        if (post_softmax)
            check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&scratch), static_cast<size_t>(rows * cols) * 8, st),
                       "alloc");
        run_threshold_f64(scores, rows, cols, theta, post_softmax, round_f32, scratch, keep, st);
        if (scratch) check_cuda(cudaFreeAsync(scratch, st), "free");
        check_cuda(cudaGetLastError(), "dsa_threshold_mask_f64");
    });
}

dsa_status dsa_sddmm_f64(int64_t rows, int64_t d, const double* q, const double* k, const uint64_t* rowptr,
                         const uint32_t* cols, int32_t scale, double* values, void* stream) {
    return guard([&] {
        require_device();
        if (rows < 0 || d < 1) throw Error(DSA_ERR_SHAPE, "sddmm: rows >= 0 and d >= 1");
        if (rows == 0) return;
        // cols / values may be null when no position is kept (nnz = 0)
        if (!q || !k || !rowptr) throw Error(DSA_ERR_PARAM, "dsa_sddmm_f64: null pointer");
        const double sc = scale ? 1.0 / std::sqrt(static_cast<double>(d)) : 1.0;  // P/src/sparse.cpp:47
        run_sddmm_f64(q, k, rowptr, cols, rows, d, sc, values, static_cast<cudaStream_t>(stream));
        check_cuda(cudaGetLastError(), "dsa_sddmm_f64");
    });
}

dsa_status dsa_sparse_softmax_f64(int64_t rows, const uint64_t* rowptr, const double* scores, double* weights,
                                  uint8_t* empty_rows, void* stream) {
    return guard([&] {
        require_device();
        if (rows < 0) throw Error(DSA_ERR_SHAPE, "sparse_softmax: rows >= 0");
        if (rows == 0) return;
        if (!rowptr) throw Error(DSA_ERR_PARAM, "dsa_sparse_softmax_f64: null pointer");
        run_sparse_softmax_f64(scores, rowptr, rows, weights, empty_rows, static_cast<cudaStream_t>(stream));
        check_cuda(cudaGetLastError(), "dsa_sparse_softmax_f64");
    });
}

dsa_status dsa_spmm_f64(int64_t rows, int64_t dv, const uint64_t* rowptr, const uint32_t* cols, const double* weights,
                        const double* v, double* z, void* stream) {
    return guard([&] {
        require_device();
        if (rows < 0 || dv < 1) throw Error(DSA_ERR_SHAPE, "spmm: rows >= 0 and d_v >= 1");
        if (rows == 0) return;
        if (!rowptr || !v || !z) throw Error(DSA_ERR_PARAM, "dsa_spmm_f64: null pointer");
        run_spmm_f64(weights, rowptr, cols, rows, v, dv, z, static_cast<cudaStream_t>(stream));
        check_cuda(cudaGetLastError(), "dsa_spmm_f64");
    });
}

int dsa_pipeline_fused(const dsa_config* cfg) {
    int out = -1;
    guard([&] {
        validate(cfg);
        const dsa_config& c = *cfg;
        if (c.mask_mode != DSA_MASK_COLVEC || pipeline_chunks(c) > 1) {
            out = 0;
            return;
        }
        dsa_mask m{};
        SelectArgs sa = select_args(c, nullptr, nullptr, nullptr, nullptr, m, Scratch{});
        out = colvec_fused_supported(sa, attn_args(c, nullptr, nullptr, nullptr, m, nullptr)) ? 1 : 0;
    });
    return out;
}

dsa_status dsa_counters(const dsa_config* cfg, const dsa_mask* mask, dsa_counts* out, void* stream) {
    return guard([&] {
        validate(cfg);
        if (!out) throw Error(DSA_ERR_PARAM, "dsa_counters: null output");
        const dsa_config& c = *cfg;
        const int64_t P = pairs_of(c);
        std::memset(out, 0, sizeof(*out));
        uint64_t nnz = 0, empty = 0;
        const double e = c.dtype == DSA_BF16 ? 2.0 : 4.0;
        switch (c.mask_mode) {
            case DSA_MASK_ROW_TOPK:
            case DSA_MASK_COLVEC: nnz = static_cast<uint64_t>(P * c.L * c.keep); break;
            case DSA_MASK_BLOCK: {
                // every kept block of block-row ib covers rows(ib) x cols(jb) positions
                if (!mask || !mask->cols) throw Error(DSA_ERR_PARAM, "dsa_counters: block mode needs the mask");
                const int64_t nb = ceil_div(c.L, c.block);
                std::vector<uint32_t> h(static_cast<size_t>(P * nb * c.keep));
                check_cuda(cudaMemcpyAsync(h.data(), mask->cols, h.size() * 4, cudaMemcpyDeviceToHost,
                                           static_cast<cudaStream_t>(stream)), "dsa_counters copy");
                check_cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "dsa_counters sync");
                for (int64_t pr = 0; pr < P; ++pr)
                    for (int64_t ib = 0; ib < nb; ++ib) {
                        const int64_t rows = std::min<int64_t>(c.block, c.L - ib * c.block);
                        for (int64_t t = 0; t < c.keep; ++t) {
                            const int64_t jb = h[(pr * nb + ib) * c.keep + t];
                            nnz += static_cast<uint64_t>(rows * std::min<int64_t>(c.block, c.L - jb * c.block));
                        }
                    }
                break;
            }
            default: {
                if (!mask || !mask->rowptr) throw Error(DSA_ERR_PARAM, "dsa_counters: threshold mode needs rowptr");
                std::vector<uint64_t> rp(static_cast<size_t>(P * c.L + 1));
                check_cuda(cudaMemcpyAsync(rp.data(), mask->rowptr, rp.size() * 8, cudaMemcpyDeviceToHost,
                                           static_cast<cudaStream_t>(stream)), "dsa_counters copy");
                check_cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "dsa_counters sync");
                nnz = rp.back();
                for (size_t r = 0; r + 1 < rp.size(); ++r) empty += rp[r + 1] == rp[r];
            }
        }
        out->nnz = nnz;
        out->sddmm_mults = nnz * static_cast<uint64_t>(c.d);
        out->spmm_mults = nnz * static_cast<uint64_t>(c.d);
        out->softmax_exps = nnz;
        out->empty_rows = empty;
        const double L = static_cast<double>(c.L);
        out->flops_predict = 4.0 * L * c.d * c.k * P;
        out->flops_score = (c.mask_mode == DSA_MASK_THRESHOLD && c.causal ? L * (L + 1) : 2.0 * L * L) * c.k * P;
        out->flops_attention = 4.0 * static_cast<double>(nnz) * c.d;
        out->bytes_predict = (2.0 * L * c.d * e + 2.0 * L * c.k * 2.0) * P + c.d * c.k * 4.0;
        out->bytes_attention = 4.0 * L * c.d * e * P;
    });
}

}  // extern "C"
