// dsattn_gpu.hpp -- C++ host mirror of the reference attention-operator API
// over the B200 C-ABI (dsa_b200.h).  Header-only; drop it into the
// reference tree next to P/include/dsattn/ and link libdsa_b200.so.
//
// Same names, value semantics and exception types as the reference:
//   dsattn::gpu::predict              <- quantize(matmul(X,P), QuantSpec)   P/include/dsattn/predictor.hpp:31-49
//   dsattn::gpu::predicted_topk_mask  <- predicted_topk_mask                P/include/dsattn/maskgen.hpp:14
//   dsattn::gpu::colvec_mask          <- colvec_mask (max-pooled bands)     P/include/dsattn/maskgen.hpp:31
//   dsattn::gpu::block_mask           <- (block extension)
//   dsattn::gpu::threshold_mask       <- threshold_mask (causal, fixed-point softmax, O6)
//   dsattn::gpu::sparse_attention     <- sddmm -> sparse_softmax -> spmm    P/include/dsattn/sparse.hpp:47-55
//   dsattn::gpu::approx_levels / predicted_topk_mask(x, PredictorParams, keep)
//                                     <- approx_scores / approx_scores_from_r (per-head W~)
//                                        P/include/dsattn/predictor.hpp:44-49, the caller's
//                                        predicted_topk_mask(approx_scores(x, pp), keep)
//                                        (P/src/trainer.cpp:162,173-175,190-195)
// The mask generators take the per-head Q and K (or X and PredictorParams)
// instead of the dense S~ the reference would materialise: S~ is computed
// exactly on the tensor cores (the integer product of the levels)
// and never leaves the GPU.  Status
// codes are rethrown as ShapeError / ParamError / ConfigError / IoError
// (P/include/dsattn/errors.hpp:9-31), so CLI exit codes are unchanged.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "dsa_b200.h"
#include "dsattn/attention.hpp"
#include "dsattn/errors.hpp"
#include "dsattn/mask.hpp"
#include "dsattn/maskgen.hpp"
#include "dsattn/matrix.hpp"
#include "dsattn/predictor.hpp"
#include "dsattn/sparse.hpp"

namespace dsattn::gpu {

[[noreturn]] inline void rethrow(dsa_status s) {
    const std::string msg = dsa_last_error();
    switch (s) {
        case DSA_ERR_SHAPE: throw ShapeError(msg);
        case DSA_ERR_PARAM: throw ParamError(msg);
        case DSA_ERR_CONFIG: throw ConfigError(msg);
        case DSA_ERR_IO: throw IoError(msg);
        case DSA_ERR_UNSUPPORTED: throw ParamError(msg);
        default: throw std::runtime_error(msg);
    }
}
inline void check(dsa_status s) {
    if (s != DSA_OK) rethrow(s);
}
inline void check_cuda(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
}

// RAII device allocation.
class DeviceBuffer {
  public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t bytes) : bytes_(bytes) {
        if (bytes) check_cuda(cudaMalloc(&p_, bytes));
    }
    ~DeviceBuffer() {
        if (p_) cudaFree(p_);
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), bytes_(o.bytes_) {
        o.p_ = nullptr;
        o.bytes_ = 0;
    }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            if (p_) cudaFree(p_);
            p_ = o.p_;
            bytes_ = o.bytes_;
            o.p_ = nullptr;
            o.bytes_ = 0;
        }
        return *this;
    }
    void* get() const { return p_; }
    size_t size() const { return bytes_; }
    template <class T>
    T* as() const {
        return static_cast<T*>(p_);
    }

  private:
    void* p_ = nullptr;
    size_t bytes_ = 0;
};

namespace detail {

inline uint16_t bf16_bits(double x) {
    float f = static_cast<float>(x);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return static_cast<uint16_t>(u >> 16);
}
inline bool bf16_exact(double x) {
    const uint16_t b = bf16_bits(x);
    uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return static_cast<double>(f) == x;
}

// The device dtype that holds every value of `ms` exactly: f32 Matrices
// -> F32; f64 Matrices of bf16 values -> BF16 (e.g. bf16 activations held in
// double); anything else -> F32 if exact, otherwise ParamError.
inline dsa_dtype pick_dtype(std::initializer_list<const Matrix*> ms) {
    bool all_bf16 = true, all_f32 = true, any_f32_prec = false;
    for (const Matrix* m : ms) {
        any_f32_prec |= m->precision() == Precision::f32;
        for (size_t i = 0; i < m->size(); ++i) {
            const double x = m->data()[i];
            all_bf16 &= bf16_exact(x);
            all_f32 &= static_cast<double>(static_cast<float>(x)) == x;
        }
    }
    if (!any_f32_prec && all_bf16) return DSA_BF16;
    if (all_f32) return DSA_F32;
    throw ParamError("dsattn::gpu: values are not exactly representable in bf16/f32");
}

inline DeviceBuffer upload(const Matrix& m, dsa_dtype dt) {
    DeviceBuffer d(m.size() * (dt == DSA_BF16 ? 2 : 4));
    if (dt == DSA_BF16) {
        std::vector<uint16_t> h(m.size());
        for (size_t i = 0; i < m.size(); ++i) h[i] = bf16_bits(m.data()[i]);
        check_cuda(cudaMemcpy(d.get(), h.data(), d.size(), cudaMemcpyHostToDevice));
    } else {
        std::vector<float> h(m.size());
        for (size_t i = 0; i < m.size(); ++i) h[i] = static_cast<float>(m.data()[i]);
        check_cuda(cudaMemcpy(d.get(), h.data(), d.size(), cudaMemcpyHostToDevice));
    }
    return d;
}

inline dsa_config base_config(const Matrix& q, const Matrix& p, int bits, dsa_dtype dt) {
    dsa_config c{};
    c.batch = 1;
    c.heads = 1;
    c.L = static_cast<int64_t>(q.rows());
    c.d = static_cast<int64_t>(q.cols());
    c.k = static_cast<int64_t>(p.cols());
    c.dtype = dt;
    c.bits = bits;
    c.quant_scope = DSA_QUANT_PER_TENSOR;
    c.round_proj_f32 = (q.precision() == Precision::f32 && p.precision() == Precision::f32) ? 1 : 0;
    c.scale = 1;
    c.keep = 1;
    c.vec_v = 8;
    c.block = 32;
    c.frac_num = 1;
    c.frac_den = 20;
    c.cap = c.L;
    return c;
}

struct DeviceLevels {
    DeviceBuffer lq, lk, sq, sk;
};

inline DeviceLevels run_predict(const dsa_config& c, const Matrix& q, const Matrix& k,
                                const Matrix& p) {
    if (q.cols() != k.cols() || q.rows() != k.rows()) throw ShapeError("predict: Q/K shapes differ");
    if (p.rows() != q.cols()) throw ShapeError("approx_scores: X feature dim != d");
    const dsa_dtype dt = static_cast<dsa_dtype>(c.dtype);
    DeviceBuffer dq = upload(q, dt), dk = upload(k, dt);
    std::vector<float> hp(p.size());
    for (size_t i = 0; i < p.size(); ++i) hp[i] = static_cast<float>(p.data()[i]);
    DeviceBuffer dp(hp.size() * 4);
    check_cuda(cudaMemcpy(dp.get(), hp.data(), dp.size(), cudaMemcpyHostToDevice));
    DeviceLevels lv;
    lv.lq = DeviceBuffer(c.L * c.k * 2);
    lv.lk = DeviceBuffer(c.L * c.k * 2);
    const size_t ns = c.quant_scope == DSA_QUANT_PER_ROW ? c.L : 1;
    lv.sq = DeviceBuffer(ns * 8);
    lv.sk = DeviceBuffer(ns * 8);
    DeviceBuffer ws(dsa_workspace_bytes(&c));
    check(dsa_predict(&c, dq.get(), dk.get(), dp.as<float>(), lv.lq.as<uint16_t>(), lv.lk.as<uint16_t>(),
                      lv.sq.as<double>(), lv.sk.as<double>(), ws.get(), ws.size(), nullptr));
    return lv;
}

inline SparseMask run_select(const dsa_config& c, const DeviceLevels& lv) {
    const int64_t cap = dsa_mask_capacity(&c);
    if (cap < 0) check(dsa_config_validate(&c));
    DeviceBuffer cols(static_cast<size_t>(cap) * 4);
    DeviceBuffer rowptr(c.mask_mode == DSA_MASK_THRESHOLD ? (c.L + 1) * 8 : 0);
    DeviceBuffer ws(dsa_workspace_bytes(&c));
    dsa_mask m{cols.as<uint32_t>(), rowptr.as<uint64_t>(), cap, nullptr};
    check(dsa_select(&c, lv.lq.as<uint16_t>(), lv.lk.as<uint16_t>(), lv.sq.as<double>(), lv.sk.as<double>(),
                     &m, ws.get(), ws.size(), nullptr));
    std::vector<uint32_t> h(static_cast<size_t>(cap));
    check_cuda(cudaMemcpy(h.data(), cols.get(), h.size() * 4, cudaMemcpyDeviceToHost));
    const size_t L = static_cast<size_t>(c.L);
    SparseMask out(L);
    switch (c.mask_mode) {
        case DSA_MASK_ROW_TOPK:
            for (size_t i = 0; i < L; ++i) out.kept[i].assign(h.begin() + i * c.keep, h.begin() + (i + 1) * c.keep);
            break;
        case DSA_MASK_COLVEC:
            for (size_t i = 0; i < L; ++i) {
                const size_t b = i / c.vec_v;
                out.kept[i].assign(h.begin() + b * c.keep, h.begin() + (b + 1) * c.keep);
            }
            break;
        case DSA_MASK_BLOCK:
            for (size_t i = 0; i < L; ++i) {
                const size_t ib = i / c.block;
                for (int64_t t = 0; t < c.keep; ++t) {
                    const size_t jb = h[ib * c.keep + t];
                    for (size_t j = jb * c.block; j < std::min(L, (jb + 1) * c.block); ++j)
                        out.kept[i].push_back(static_cast<uint32_t>(j));
                }
            }
            break;
        default: {
            std::vector<uint64_t> rp(L + 1);
            check_cuda(cudaMemcpy(rp.data(), rowptr.get(), rp.size() * 8, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < L; ++i) out.kept[i].assign(h.begin() + rp[i], h.begin() + rp[i + 1]);
        }
    }
    return out;
}

inline DeviceBuffer upload_f64(const Matrix& m) {
    DeviceBuffer d(m.size() * 8);
    check_cuda(cudaMemcpy(d.get(), m.data(), d.size(), cudaMemcpyHostToDevice));
    return d;
}

// approx_scores / approx_scores_from_r levels on the device (x or r given).
inline DeviceLevels run_predict_wtilde(const dsa_config& c, const Matrix* x, const Matrix* r,
                                       const PredictorParams& pp) {
    pp.validate();
    const Matrix& P = pp.proj->p;
    DeviceBuffer dx, dp, dr(static_cast<size_t>(c.L * c.k) * 8);
    if (x) {
        if (x->cols() != P.rows()) throw ShapeError("approx_scores: X feature dim != d");
        dx = upload_f64(*x);
        dp = upload_f64(P);
    } else {
        if (r->cols() != P.cols()) throw ShapeError("approx_scores: R width != projection k");
        dr = upload_f64(*r);
    }
    DeviceBuffer dwq = upload_f64(pp.wq), dwk = upload_f64(pp.wk);
    DeviceLevels lv;
    lv.lq = DeviceBuffer(static_cast<size_t>(c.L * c.k) * 2);
    lv.lk = DeviceBuffer(static_cast<size_t>(c.L * c.k) * 2);
    const size_t ns = c.quant_scope == DSA_QUANT_PER_ROW ? static_cast<size_t>(c.L) : 1;
    lv.sq = DeviceBuffer(ns * 8);
    lv.sk = DeviceBuffer(ns * 8);
    DeviceBuffer ws(dsa_predict_wtilde_workspace_bytes(&c));
    check(dsa_predict_wtilde(&c, x ? static_cast<int64_t>(x->cols()) : 0, x ? dx.as<double>() : nullptr,
                             x ? dp.as<double>() : nullptr, dr.as<double>(), dwq.as<double>(), dwk.as<double>(),
                             lv.lq.as<uint16_t>(), lv.lk.as<uint16_t>(), lv.sq.as<double>(), lv.sk.as<double>(),
                             ws.get(), ws.size(), nullptr));
    return lv;
}

// Does the reference round the predictor's matmuls to f32?  A product is
// f32 only when BOTH operands are (combine(), P/include/dsattn/matrix.hpp:
// 90-93): R = X P rounds iff X and P are f32, R W~ rounds iff R and W~ are.
// The device chain has one switch for both stages (round_proj_f32), so the
// answer is true when every operand is f32, false when the chain is f64
// from its first product on (X or P f64 -- the ToyModel case: f32 weights,
// f64 ternary P -- or a given R that is f64 or meets f64 W~), and the one
// remaining mix (stage one rounds, stage two does not, or W~_Q and W~_K
// differ) is rejected.  `x`/`p` are null when R is given.
inline bool chain_f32(const Matrix* x, const Matrix* p, const Matrix* r, const Matrix& wq, const Matrix& wk) {
    const auto f32 = [](const Matrix& m) { return m.precision() == Precision::f32; };
    const bool r32 = r ? f32(*r) : (f32(*x) && f32(*p));
    if (f32(wq) != f32(wk))
        throw ParamError("dsattn::gpu: W~_Q and W~_K of different precisions are not supported");
    const bool s32 = r32 && f32(wq);
    if (!r && r32 && !s32)
        throw ParamError("dsattn::gpu: mixed f32/f64 predictor operands are not supported");
    return s32;
}

inline dsa_config wtilde_config(size_t L, const PredictorParams& pp, bool f32) {
    dsa_config c{};
    c.batch = c.heads = 1;
    c.L = static_cast<int64_t>(L);
    c.d = 64;  // unused by the predictor; a valid head width for dsa_config_validate
    c.k = static_cast<int64_t>(pp.proj->p.cols());
    c.dtype = DSA_BF16;
    c.bits = pp.quant.bits;
    c.quant_scope = DSA_QUANT_PER_TENSOR;
    c.round_proj_f32 = f32 ? 1 : 0;
    c.scale = 1;
    c.keep = 1;
    c.vec_v = 8;
    c.block = 32;
    c.frac_num = 1;
    c.frac_den = 20;
    c.cap = c.L;
    return c;
}

inline Matrix levels_to_matrix(const DeviceBuffer& d, size_t L, size_t K) {
    std::vector<uint16_t> h(L * K);
    check_cuda(cudaMemcpy(h.data(), d.get(), h.size() * 2, cudaMemcpyDeviceToHost));
    Matrix m(L, K);
    for (size_t r = 0; r < L; ++r)
        for (size_t c = 0; c < K; ++c) {  // chunk-planar [K/8][L][8] -> row-major
            uint32_t u = static_cast<uint32_t>(h[((c / 8) * L + r) * 8 + c % 8]) << 16;
            float f;
            std::memcpy(&f, &u, 4);
            m.raw()[r * K + c] = f;
        }
    return m;
}

}  // namespace detail

// Integer levels (held exactly in f64 Matrices) and scales of quant(Q.P),
// quant(K.P).  Per-tensor scope is the reference's (predictor.cpp:37-41).
struct Levels {
    Matrix q, k;
    std::vector<double> scale_q, scale_k;
};

inline Levels predict(const Matrix& q, const Matrix& k, const Matrix& p, QuantSpec quant,
                      bool per_row = false) {
    quant.validate();
    const dsa_dtype dt = detail::pick_dtype({&q, &k});
    dsa_config c = detail::base_config(q, p, quant.bits, dt);
    c.quant_scope = per_row ? DSA_QUANT_PER_ROW : DSA_QUANT_PER_TENSOR;
    check(dsa_config_validate(&c));
    detail::DeviceLevels lv = detail::run_predict(c, q, k, p);
    Levels out{Matrix(q.rows(), p.cols()), Matrix(k.rows(), p.cols()), {}, {}};
    std::vector<uint16_t> h(q.rows() * p.cols());
    for (int w = 0; w < 2; ++w) {
        check_cuda(cudaMemcpy(h.data(), (w ? lv.lk : lv.lq).get(), h.size() * 2, cudaMemcpyDeviceToHost));
        Matrix& m = w ? out.k : out.q;
        const size_t L = q.rows(), K = p.cols();
        for (size_t r = 0; r < L; ++r)
            for (size_t c = 0; c < K; ++c) {  // chunk-planar [K/8][L][8] -> row-major
                uint32_t u = static_cast<uint32_t>(h[((c / 8) * L + r) * 8 + c % 8]) << 16;
                float f;
                std::memcpy(&f, &u, 4);
                m.raw()[r * K + c] = f;
            }
        std::vector<double>& s = w ? out.scale_k : out.scale_q;
        s.resize(per_row ? q.rows() : 1);
        check_cuda(cudaMemcpy(s.data(), (w ? lv.sk : lv.sq).get(), s.size() * 8, cudaMemcpyDeviceToHost));
    }
    return out;
}

// approx_scores(x, pp) / approx_scores_from_r(r, pp) (P/src/predictor.cpp:
// 67-80) as exact integer levels + per-tensor scales: R = X P, Q~ =
// quantize(R W~_Q), K~ = quantize(R W~_K) -- bit-identical to the
// reference's (fp64 chains on the device; f32 when every operand is f32).
// S~ = s_q s_k (levels_q levels_k^T).
inline Levels approx_levels(const Matrix& x, const PredictorParams& pp) {
    const bool f32 = detail::chain_f32(&x, &pp.proj->p, nullptr, pp.wq, pp.wk);
    dsa_config c = detail::wtilde_config(x.rows(), pp, f32);
    check(dsa_config_validate(&c));
    detail::DeviceLevels lv = detail::run_predict_wtilde(c, &x, nullptr, pp);
    Levels out{detail::levels_to_matrix(lv.lq, x.rows(), c.k), detail::levels_to_matrix(lv.lk, x.rows(), c.k),
               std::vector<double>(1), std::vector<double>(1)};
    check_cuda(cudaMemcpy(out.scale_q.data(), lv.sq.get(), 8, cudaMemcpyDeviceToHost));
    check_cuda(cudaMemcpy(out.scale_k.data(), lv.sk.get(), 8, cudaMemcpyDeviceToHost));
    return out;
}

// The reference caller's predicted mask, predicted_topk_mask(approx_scores(x,
// pp), keep) (P/src/trainer.cpp:190-195), ranked on the exact integer S~
// (ties to the lowest column).
inline SparseMask predicted_topk_mask(const Matrix& x, const PredictorParams& pp, size_t keep_per_row) {
    const bool f32 = detail::chain_f32(&x, &pp.proj->p, nullptr, pp.wq, pp.wk);
    dsa_config c = detail::wtilde_config(x.rows(), pp, f32);
    c.mask_mode = DSA_MASK_ROW_TOPK;
    c.keep = static_cast<int64_t>(keep_per_row);
    check(dsa_config_validate(&c));
    return detail::run_select(c, detail::run_predict_wtilde(c, &x, nullptr, pp));
}

// Same from a precomputed R = X P (approx_scores_from_r).
inline SparseMask predicted_topk_mask_from_r(const Matrix& r, const PredictorParams& pp, size_t keep_per_row) {
    const bool f32 = detail::chain_f32(nullptr, nullptr, &r, pp.wq, pp.wk);
    dsa_config c = detail::wtilde_config(r.rows(), pp, f32);
    c.mask_mode = DSA_MASK_ROW_TOPK;
    c.keep = static_cast<int64_t>(keep_per_row);
    check(dsa_config_validate(&c));
    return detail::run_select(c, detail::run_predict_wtilde(c, nullptr, &r, pp));
}

inline SparseMask predicted_topk_mask(const Matrix& q, const Matrix& k, const Matrix& p,
                                      QuantSpec quant, size_t keep_per_row, bool per_row = false) {
    quant.validate();
    dsa_config c = detail::base_config(q, p, quant.bits, detail::pick_dtype({&q, &k}));
    c.quant_scope = per_row ? DSA_QUANT_PER_ROW : DSA_QUANT_PER_TENSOR;
    c.mask_mode = DSA_MASK_ROW_TOPK;
    c.keep = static_cast<int64_t>(keep_per_row);
    check(dsa_config_validate(&c));
    return detail::run_select(c, detail::run_predict(c, q, k, p));
}

inline SparseMask colvec_mask(const Matrix& q, const Matrix& k, const Matrix& p, QuantSpec quant,
                              ColVecSpec spec, size_t keep_per_band) {
    quant.validate();
    if (spec.orientation != VecOrientation::col)
        throw ParamError("dsattn::gpu::colvec_mask: only column vectors (v query rows x 1 key)");
    dsa_config c = detail::base_config(q, p, quant.bits, detail::pick_dtype({&q, &k}));
    c.mask_mode = DSA_MASK_COLVEC;
    c.vec_v = static_cast<int32_t>(spec.v);
    c.keep = static_cast<int64_t>(keep_per_band);
    check(dsa_config_validate(&c));
    return detail::run_select(c, detail::run_predict(c, q, k, p));
}

inline SparseMask block_mask(const Matrix& q, const Matrix& k, const Matrix& p, QuantSpec quant,
                             size_t block, size_t keep_blocks, bool force_diag) {
    quant.validate();
    dsa_config c = detail::base_config(q, p, quant.bits, detail::pick_dtype({&q, &k}));
    c.mask_mode = DSA_MASK_BLOCK;
    c.block = static_cast<int32_t>(block);
    c.keep = static_cast<int64_t>(keep_blocks);
    c.force_diag = force_diag ? 1 : 0;
    check(dsa_config_validate(&c));
    return detail::run_select(c, detail::run_predict(c, q, k, p));
}

// Keeps p~ >= frac_den / (frac_num * L) of softmax(s_q s_k S_int / sqrt(d))
// (causal: over j <= i), at most `cap` per row; rows may be empty.
inline SparseMask threshold_mask(const Matrix& q, const Matrix& k, const Matrix& p, QuantSpec quant,
                                 int64_t frac_num, int64_t frac_den, size_t cap, bool causal) {
    quant.validate();
    dsa_config c = detail::base_config(q, p, quant.bits, detail::pick_dtype({&q, &k}));
    c.mask_mode = DSA_MASK_THRESHOLD;
    c.frac_num = frac_num;
    c.frac_den = frac_den;
    c.cap = static_cast<int64_t>(cap);
    c.causal = causal ? 1 : 0;
    check(dsa_config_validate(&c));
    return detail::run_select(c, detail::run_predict(c, q, k, p));
}

namespace detail {

// The densest device layout a reference SparseMask fits (dsa_mask, dsa_b200.h):
//   COLVEC   every 8-row band shares one list (band-shared tensor-core tiles)
//   BLOCK    32 x 32 blocks: every 32-row block row shares a list that is a
//            union of whole, aligned 32-column blocks (L % 32 == 0)
//   ROW_TOPK every row keeps the same number of keys
//   THRESHOLD (CSR) anything else (ragged rows, empty rows)
struct MaskLayout {
    dsa_mask_mode mode;
    int64_t keep;
    std::vector<uint32_t> cols;
    std::vector<uint64_t> rowptr;
};

inline MaskLayout layout_of(const SparseMask& m) {
    const size_t L = m.l;
    MaskLayout out{DSA_MASK_THRESHOLD, 0, {}, {}};
    bool uniform = L > 0 && !m.kept[0].empty();
    for (size_t i = 1; i < L && uniform; ++i) uniform = m.kept[i].size() == m.kept[0].size();
    if (uniform) {
        const size_t n = m.kept[0].size();
        bool bands = true;
        for (size_t i = 0; i < L && bands; ++i) bands = m.kept[i] == m.kept[i - i % 8];
        bool blocks = L % 32 == 0 && n % 32 == 0;
        for (size_t i = 0; i < L && blocks; ++i) blocks = m.kept[i] == m.kept[i - i % 32];
        for (size_t i = 0; i < L && blocks; i += 32)
            for (size_t t = 0; t < n && blocks; ++t)
                blocks = m.kept[i][t] == m.kept[i][t - t % 32] + t % 32 && m.kept[i][t - t % 32] % 32 == 0;
        if (blocks) {
            out.mode = DSA_MASK_BLOCK;
            out.keep = static_cast<int64_t>(n / 32);
            for (size_t i = 0; i < L; i += 32)
                for (size_t t = 0; t < n; t += 32) out.cols.push_back(m.kept[i][t] / 32);
        } else if (bands) {
            out.mode = DSA_MASK_COLVEC;
            out.keep = static_cast<int64_t>(n);
            for (size_t i = 0; i < L; i += 8) out.cols.insert(out.cols.end(), m.kept[i].begin(), m.kept[i].end());
        } else {
            out.mode = DSA_MASK_ROW_TOPK;
            out.keep = static_cast<int64_t>(n);
            for (size_t i = 0; i < L; ++i) out.cols.insert(out.cols.end(), m.kept[i].begin(), m.kept[i].end());
        }
        return out;
    }
    out.rowptr.assign(L + 1, 0);
    for (size_t i = 0; i < L; ++i) {
        out.rowptr[i + 1] = out.rowptr[i] + m.kept[i].size();
        out.cols.insert(out.cols.end(), m.kept[i].begin(), m.kept[i].end());
    }
    return out;
}

}  // namespace detail

// sddmm -> sparse_softmax -> spmm for one head; empty rows give zero rows
// (flagged in *empty_rows when given).  Output precision follows V.  The
// mask is routed by its structure (detail::layout_of): band-shared and
// block masks reach the tensor-core band / block kernels, uniform rows the
// row-list layout, everything else the CSR layout.
inline Matrix sparse_attention(const Matrix& q, const Matrix& k, const Matrix& v,
                               const SparseMask& mask, bool scale,
                               std::vector<uint8_t>* empty_rows = nullptr) {
    if (q.cols() != k.cols()) throw ShapeError("sddmm: Q/K feature dims differ");
    if (q.rows() != mask.l || k.rows() != mask.l) throw ShapeError("sddmm: mask size != sequence length");
    if (v.rows() != mask.l) throw ShapeError("spmm: V rows != sequence length");
    if (v.cols() != q.cols()) throw ShapeError("dsattn::gpu: needs d_v == d_k");
    mask.validate();
    const dsa_dtype dt = detail::pick_dtype({&q, &k, &v});
    const detail::MaskLayout ml = detail::layout_of(mask);
    dsa_config c{};
    c.batch = c.heads = 1;
    c.L = static_cast<int64_t>(q.rows());
    c.d = static_cast<int64_t>(q.cols());
    c.k = 16;
    c.dtype = dt;
    c.bits = 4;
    c.mask_mode = ml.mode;
    c.keep = std::max<int64_t>(ml.keep, 1);
    c.vec_v = 8;
    c.block = 32;
    c.scale = scale ? 1 : 0;
    c.frac_num = 1;
    c.frac_den = 1;
    c.cap = c.L;
    check(dsa_config_validate(&c));
    DeviceBuffer dq = detail::upload(q, dt), dk = detail::upload(k, dt), dv = detail::upload(v, dt);
    DeviceBuffer dz(dq.size()), drp(std::max<size_t>(ml.rowptr.size(), 1) * 8),
        dc(std::max<size_t>(ml.cols.size(), 1) * 4), de(mask.l);
    if (!ml.rowptr.empty())
        check_cuda(cudaMemcpy(drp.get(), ml.rowptr.data(), ml.rowptr.size() * 8, cudaMemcpyHostToDevice));
    if (!ml.cols.empty())
        check_cuda(cudaMemcpy(dc.get(), ml.cols.data(), ml.cols.size() * 4, cudaMemcpyHostToDevice));
    if (ml.mode != DSA_MASK_THRESHOLD) check_cuda(cudaMemset(de.get(), 0, mask.l));
    dsa_mask m{dc.as<uint32_t>(), ml.rowptr.empty() ? nullptr : drp.as<uint64_t>(),
               static_cast<int64_t>(ml.cols.size()), de.as<uint8_t>()};
    check(dsa_sparse_attention(&c, dq.get(), dk.get(), dv.get(), &m, dz.get(), nullptr));
    Matrix z(mask.l, v.cols(), v.precision());
    if (dt == DSA_BF16) {
        std::vector<uint16_t> h(z.size());
        check_cuda(cudaMemcpy(h.data(), dz.get(), h.size() * 2, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < h.size(); ++i) {
            uint32_t u = static_cast<uint32_t>(h[i]) << 16;
            float f;
            std::memcpy(&f, &u, 4);
            z.raw()[i] = f;
        }
    } else {
        std::vector<float> h(z.size());
        check_cuda(cudaMemcpy(h.data(), dz.get(), h.size() * 4, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < h.size(); ++i) z.raw()[i] = h[i];
    }
    z.round_to_precision();
    if (empty_rows) {
        empty_rows->resize(mask.l);
        check_cuda(cudaMemcpy(empty_rows->data(), de.get(), mask.l, cudaMemcpyDeviceToHost));
    }
    return z;
}

namespace detail {
inline void csr_of(const SparseMask& mask, std::vector<uint64_t>& rowptr, std::vector<uint32_t>& cols) {
    rowptr.assign(mask.l + 1, 0);
    cols.clear();
    for (size_t i = 0; i < mask.l; ++i) {
        cols.insert(cols.end(), mask.kept[i].begin(), mask.kept[i].end());
        rowptr[i + 1] = cols.size();
    }
}
inline DeviceBuffer upload_raw(const void* p, size_t bytes) {
    DeviceBuffer d(std::max<size_t>(bytes, 8));
    if (bytes) check_cuda(cudaMemcpy(d.get(), p, bytes, cudaMemcpyHostToDevice));
    return d;
}
}  // namespace detail

// row_topk_indices (P/src/linalg.cpp:69-85) and oracle_topk_mask
// (P/src/maskgen.cpp:11-16) on a score matrix the caller holds: value
// descending, the lowest column among equals, ascending lists -- identical
// to the reference for every input without NaNs.
inline std::vector<std::vector<uint32_t>> row_topk_indices(const Matrix& s, size_t k_keep) {
    if (k_keep < 1 || k_keep > s.cols()) throw ParamError("row_topk_indices: k_keep out of range");
    DeviceBuffer ds = detail::upload_f64(s), dout(s.rows() * k_keep * 4);
    check(dsa_row_topk_f64(static_cast<int64_t>(s.rows()), static_cast<int64_t>(s.cols()), ds.as<double>(),
                           static_cast<int64_t>(k_keep), dout.as<uint32_t>(), nullptr));
    std::vector<uint32_t> flat(s.rows() * k_keep);
    check_cuda(cudaMemcpy(flat.data(), dout.get(), flat.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<std::vector<uint32_t>> out(s.rows());
    for (size_t i = 0; i < s.rows(); ++i) out[i].assign(flat.begin() + i * k_keep, flat.begin() + (i + 1) * k_keep);
    return out;
}

inline SparseMask oracle_topk_mask(const Matrix& s, size_t keep_per_row) {
    if (s.rows() != s.cols()) throw ShapeError("oracle_topk_mask: scores must be square");
    SparseMask m(s.rows());
    m.kept = gpu::row_topk_indices(s, keep_per_row);
    return m;
}

// colvec_mask and threshold_mask with the reference's OWN signatures, on a
// dense score matrix the caller holds (P/include/dsattn/maskgen.hpp:14-30,
// P/src/maskgen.cpp:22-61): the band rule is the reference's sum of |s~| over
// the band, keep = ceil((1 - sparsity) l); row orientation is the transposed
// rule.  (The (q, k, p, quant) overloads above never materialise S~ and apply
// the BASELINE max-pooled integer rule.)
inline SparseMask colvec_mask(const Matrix& s_tilde, ColVecSpec spec, double target_sparsity) {
    if (spec.orientation == VecOrientation::row) {
        ColVecSpec t = spec;
        t.orientation = VecOrientation::col;
        Matrix tr(s_tilde.cols(), s_tilde.rows(), s_tilde.precision());
        for (size_t i = 0; i < s_tilde.rows(); ++i)
            for (size_t j = 0; j < s_tilde.cols(); ++j) tr.raw()[j * s_tilde.rows() + i] = s_tilde(i, j);
        SparseMask cm = gpu::colvec_mask(tr, t, target_sparsity);
        SparseMask m(cm.l);
        for (size_t i = 0; i < cm.l; ++i)
            for (uint32_t j : cm.kept[i]) m.kept[j].push_back(static_cast<uint32_t>(i));
        return m;
    }
    if (spec.v < 1) throw ParamError("colvec_mask: vector height must be >= 1");
    if (!(target_sparsity > 0.0 && target_sparsity < 1.0))
        throw ParamError("colvec_mask: target_sparsity must be in (0, 1)");
    if (s_tilde.rows() != s_tilde.cols()) throw ShapeError("colvec_mask: scores must be square");
    const size_t l = s_tilde.rows();
    const auto keep = static_cast<size_t>(std::ceil((1.0 - target_sparsity) * static_cast<double>(l)));
    const size_t nb = (l + spec.v - 1) / spec.v;
    DeviceBuffer ds = detail::upload_f64(s_tilde), dout(nb * keep * 4);
    check(dsa_colvec_mask_f64(static_cast<int64_t>(l), static_cast<int64_t>(spec.v), static_cast<int64_t>(keep),
                              ds.as<double>(), dout.as<uint32_t>(), nullptr));
    std::vector<uint32_t> flat(nb * keep);
    check_cuda(cudaMemcpy(flat.data(), dout.get(), flat.size() * 4, cudaMemcpyDeviceToHost));
    SparseMask m(l);
    for (size_t i = 0; i < l; ++i) {
        const size_t b = i / spec.v;
        m.kept[i].assign(flat.begin() + b * keep, flat.begin() + (b + 1) * keep);
    }
    return m;
}

inline SparseMask threshold_mask(const Matrix& s, double theta, bool post_softmax) {
    if (!std::isfinite(theta)) throw ParamError("threshold_mask: theta must be finite");
    if (s.rows() != s.cols()) throw ShapeError("threshold_mask: scores must be square");
    const size_t l = s.rows();
    DeviceBuffer ds = detail::upload_f64(s), dk(l * l);
    check(dsa_threshold_mask_f64(static_cast<int64_t>(l), static_cast<int64_t>(l), ds.as<double>(), theta,
                                 post_softmax ? 1 : 0, s.precision() == Precision::f32 ? 1 : 0, dk.as<uint8_t>(),
                                 nullptr));
    std::vector<uint8_t> keep(l * l);
    check_cuda(cudaMemcpy(keep.data(), dk.get(), keep.size(), cudaMemcpyDeviceToHost));
    SparseMask m(l);
    for (size_t i = 0; i < l; ++i)
        for (uint32_t j = 0; j < l; ++j)
            if (keep[i * l + j]) m.kept[i].push_back(j);
    return m;
}

// prediction_accuracy (P/src/maskgen.cpp:94-107) on the device: the fraction
// of predicted positions the oracle mask also keeps (dsa_prediction_accuracy
// over both masks' CSR); the reference's ParamErrors for a size mismatch,
// unequal per-row counts and empty masks.
inline double prediction_accuracy(const SparseMask& pred, const SparseMask& oracle) {
    if (pred.l != oracle.l) throw ParamError("prediction_accuracy: size mismatch");
    std::vector<uint64_t> rp, ro;
    std::vector<uint32_t> cp, co;
    detail::csr_of(pred, rp, cp);
    detail::csr_of(oracle, ro, co);
    if (pred.l == 0 || cp.empty()) {
        for (size_t i = 0; i < pred.l; ++i)
            if (pred.kept[i].size() != oracle.kept[i].size())
                throw ParamError("prediction_accuracy: per-row counts differ");
        throw ParamError("prediction_accuracy: empty masks");
    }
    dsa_config c{};
    c.batch = c.heads = 1;
    c.L = static_cast<int64_t>(pred.l);
    c.d = 64;
    c.k = 16;
    c.dtype = DSA_BF16;
    c.bits = 4;
    c.mask_mode = DSA_MASK_THRESHOLD;  // general CSR
    c.scale = 1;
    c.keep = 1;
    c.vec_v = 8;
    c.block = 32;
    c.frac_num = c.frac_den = 1;
    c.cap = c.L;
    check(dsa_config_validate(&c));
    DeviceBuffer drp = detail::upload_raw(rp.data(), rp.size() * 8), dcp = detail::upload_raw(cp.data(), cp.size() * 4),
                 dro = detail::upload_raw(ro.data(), ro.size() * 8), dco = detail::upload_raw(co.data(), co.size() * 4);
    dsa_mask mp{dcp.as<uint32_t>(), drp.as<uint64_t>(), static_cast<int64_t>(cp.size()), nullptr};
    dsa_mask mo{dco.as<uint32_t>(), dro.as<uint64_t>(), static_cast<int64_t>(co.size()), nullptr};
    double acc = 0.0;
    check(dsa_prediction_accuracy(&c, &mp, &mo, &acc, nullptr));
    return acc;
}

// The three operators separately, as the reference exposes them
// (P/include/dsattn/sparse.hpp:47-55): same types, same exceptions, f64
// values.  sddmm and spmm reproduce the reference's scalar kernels bit for
// bit (one fma per term in index order), sparse_softmax to the last ulp of
// exp().  The fused sparse_attention above is the hot path; these are for
// callers that inspect the scores or weights in between.

inline SparseScores sddmm(const Matrix& q, const Matrix& k, const SparseMask& mask, bool scale) {
    if (q.cols() != k.cols()) throw ShapeError("sddmm: Q/K feature dims differ");
    if (q.rows() != mask.l || k.rows() != mask.l) throw ShapeError("sddmm: mask size != sequence length");
    mask.validate();
    SparseScores out;
    out.mask = mask;
    std::vector<uint32_t> cols;
    detail::csr_of(mask, out.row_offsets, cols);
    out.values.resize(cols.size());
    DeviceBuffer dq = detail::upload_f64(q), dk = detail::upload_f64(k),
                 drp = detail::upload_raw(out.row_offsets.data(), out.row_offsets.size() * 8),
                 dc = detail::upload_raw(cols.data(), cols.size() * 4), dv(std::max<size_t>(cols.size(), 1) * 8);
    check(dsa_sddmm_f64(static_cast<int64_t>(mask.l), static_cast<int64_t>(q.cols()), dq.as<double>(), dk.as<double>(),
                        drp.as<uint64_t>(), dc.as<uint32_t>(), scale ? 1 : 0, dv.as<double>(), nullptr));
    if (!cols.empty())
        check_cuda(cudaMemcpy(out.values.data(), dv.get(), cols.size() * 8, cudaMemcpyDeviceToHost));
    else
        check_cuda(cudaDeviceSynchronize());
    return out;
}

inline SparseWeights sparse_softmax(const SparseScores& s) {
    SparseWeights out;
    out.mask = s.mask;
    out.row_offsets = s.row_offsets;
    out.values.resize(s.values.size());
    out.empty_row.assign(s.mask.l, 0);
    if (s.mask.l == 0) return out;
    DeviceBuffer drp = detail::upload_raw(s.row_offsets.data(), s.row_offsets.size() * 8),
                 ds = detail::upload_raw(s.values.data(), s.values.size() * 8),
                 dw(std::max<size_t>(s.values.size(), 1) * 8), de(s.mask.l);
    check(dsa_sparse_softmax_f64(static_cast<int64_t>(s.mask.l), drp.as<uint64_t>(), ds.as<double>(), dw.as<double>(),
                                 de.as<uint8_t>(), nullptr));
    if (!s.values.empty())
        check_cuda(cudaMemcpy(out.values.data(), dw.get(), s.values.size() * 8, cudaMemcpyDeviceToHost));
    check_cuda(cudaMemcpy(out.empty_row.data(), de.get(), s.mask.l, cudaMemcpyDeviceToHost));
    return out;
}

inline Matrix spmm(const SparseWeights& a, const Matrix& v) {
    if (a.mask.l != v.rows()) throw ShapeError("spmm: V rows != sequence length");
    Matrix z(a.mask.l, v.cols(), v.precision());
    if (z.size() == 0) return z;
    std::vector<uint32_t> cols;
    cols.reserve(a.values.size());
    for (const auto& row : a.mask.kept) cols.insert(cols.end(), row.begin(), row.end());
    DeviceBuffer drp = detail::upload_raw(a.row_offsets.data(), a.row_offsets.size() * 8),
                 dc = detail::upload_raw(cols.data(), cols.size() * 4),
                 dw = detail::upload_raw(a.values.data(), a.values.size() * 8), dv = detail::upload_f64(v),
                 dz(z.size() * 8);
    check(dsa_spmm_f64(static_cast<int64_t>(a.mask.l), static_cast<int64_t>(v.cols()), drp.as<uint64_t>(),
                       dc.as<uint32_t>(), dw.as<double>(), dv.as<double>(), dz.as<double>(), nullptr));
    check_cuda(cudaMemcpy(z.raw(), dz.get(), z.size() * 8, cudaMemcpyDeviceToHost));
    z.round_to_precision();
    return z;
}

// project_qkv (P/src/attention.cpp:36-46) on the tensor cores: every head's
// Q, K, V in one bf16 GEMM over X (dsa_project_qkv).  X and the weights are
// rounded to bf16 (exact when they already are), products accumulate in
// fp32 and the outputs are rounded to bf16 -- the BASELINE bf16 tolerance,
// not the reference's f64.  Same signature, value semantics and exceptions.
inline Qkv project_qkv(const Matrix& x, const AttentionParams& p) {
    p.validate();
    if (x.cols() != p.d()) throw ShapeError("project_qkv: X feature dim != d");
    const int64_t L = static_cast<int64_t>(x.rows()), dm = static_cast<int64_t>(p.d());
    const int64_t H = static_cast<int64_t>(p.heads), dk = static_cast<int64_t>(p.d_k()),
                  dv = static_cast<int64_t>(p.d_v());
    const int64_t n_out = H * (2 * dk + dv);
    std::vector<uint16_t> hx(x.size()), hw(static_cast<size_t>(n_out * dm));
    for (size_t i = 0; i < x.size(); ++i) hx[i] = detail::bf16_bits(x.data()[i]);
    int64_t row = 0;
    auto pack = [&](const std::vector<Matrix>& ws) {
        for (const Matrix& w : ws)
            for (size_t c = 0; c < w.cols(); ++c, ++row)
                for (size_t r = 0; r < w.rows(); ++r) hw[static_cast<size_t>(row * dm) + r] = detail::bf16_bits(w(r, c));
    };
    pack(p.wq);
    pack(p.wk);
    pack(p.wv);
    DeviceBuffer dx(hx.size() * 2), dw(hw.size() * 2), dq(static_cast<size_t>(H * L * dk) * 2),
        dkb(static_cast<size_t>(H * L * dk) * 2), dvb(static_cast<size_t>(H * L * dv) * 2);
    check_cuda(cudaMemcpy(dx.get(), hx.data(), dx.size(), cudaMemcpyHostToDevice));
    check_cuda(cudaMemcpy(dw.get(), hw.data(), dw.size(), cudaMemcpyHostToDevice));
    check(dsa_project_qkv(1, L, dm, H, dk, dv, 0, dx.get(), dw.get(), dq.get(), dkb.get(), dvb.get(), nullptr,
                          nullptr));
    auto fetch = [&](const DeviceBuffer& d, int64_t cols) {
        std::vector<uint16_t> h(static_cast<size_t>(H * L * cols));
        check_cuda(cudaMemcpy(h.data(), d.get(), h.size() * 2, cudaMemcpyDeviceToHost));
        std::vector<Matrix> out;
        for (int64_t hd = 0; hd < H; ++hd) {
            Matrix m(static_cast<size_t>(L), static_cast<size_t>(cols), x.precision());
            for (int64_t i = 0; i < L * cols; ++i) {
                uint32_t u = static_cast<uint32_t>(h[static_cast<size_t>(hd * L * cols + i)]) << 16;
                float f;
                std::memcpy(&f, &u, 4);
                m.raw()[static_cast<size_t>(i)] = f;
            }
            m.round_to_precision();
            out.push_back(std::move(m));
        }
        return out;
    };
    Qkv out;
    out.q = fetch(dq, dk);
    out.k = fetch(dkb, dk);
    out.v = fetch(dvb, dv);
    return out;
}

// sparse_attention(x, params, per-head masks) (P/src/sparse.cpp:93-120): the
// layer-level composition -- project_qkv for every head in one tensor-core
// GEMM (device-resident Q/K/V, bf16), then SDDMM -> sparse softmax -> SpMM
// for all heads in one batched call over the heads' masks, heads
// concatenated by columns.  Needs d_v == d_k.
inline Matrix sparse_attention(const Matrix& x, const AttentionParams& p, std::span<const SparseMask> per_head) {
    if (per_head.size() != p.heads) throw ShapeError("sparse_attention: need one mask per head");
    p.validate();
    if (x.cols() != p.d()) throw ShapeError("project_qkv: X feature dim != d");
    const int64_t L = static_cast<int64_t>(x.rows()), dm = static_cast<int64_t>(p.d());
    const int64_t H = static_cast<int64_t>(p.heads), dk = static_cast<int64_t>(p.d_k()),
                  dv = static_cast<int64_t>(p.d_v());
    if (dk != dv) throw ShapeError("dsattn::gpu: needs d_v == d_k");
    std::vector<uint64_t> rp(static_cast<size_t>(H * L) + 1, 0);
    std::vector<uint32_t> cols;
    for (int64_t h = 0; h < H; ++h) {
        const SparseMask& m = per_head[static_cast<size_t>(h)];
        if (m.l != static_cast<size_t>(L)) throw ShapeError("sddmm: mask size != sequence length");
        m.validate();
        for (int64_t i = 0; i < L; ++i) {
            const auto& row = m.kept[static_cast<size_t>(i)];
            rp[static_cast<size_t>(h * L + i) + 1] = rp[static_cast<size_t>(h * L + i)] + row.size();
            cols.insert(cols.end(), row.begin(), row.end());
        }
    }
    std::vector<uint16_t> hx(x.size()), hw(static_cast<size_t>(H * (2 * dk + dv) * dm));
    for (size_t i = 0; i < x.size(); ++i) hx[i] = detail::bf16_bits(x.data()[i]);
    int64_t row = 0;
    for (const auto* ws : {&p.wq, &p.wk, &p.wv})
        for (const Matrix& w : *ws)
            for (size_t c = 0; c < w.cols(); ++c, ++row)
                for (size_t r = 0; r < w.rows(); ++r) hw[static_cast<size_t>(row * dm) + r] = detail::bf16_bits(w(r, c));
    const size_t nqkv = static_cast<size_t>(H * L * dk) * 2;
    DeviceBuffer dx(hx.size() * 2), dw(hw.size() * 2), dq(nqkv), dkb(nqkv), dvb(nqkv), dz(nqkv), drp(rp.size() * 8),
        dc(std::max<size_t>(cols.size(), 1) * 4);
    check_cuda(cudaMemcpy(dx.get(), hx.data(), dx.size(), cudaMemcpyHostToDevice));
    check_cuda(cudaMemcpy(dw.get(), hw.data(), dw.size(), cudaMemcpyHostToDevice));
    check_cuda(cudaMemcpy(drp.get(), rp.data(), drp.size(), cudaMemcpyHostToDevice));
    if (!cols.empty()) check_cuda(cudaMemcpy(dc.get(), cols.data(), cols.size() * 4, cudaMemcpyHostToDevice));
    check(dsa_project_qkv(1, L, dm, H, dk, dv, 0, dx.get(), dw.get(), dq.get(), dkb.get(), dvb.get(), nullptr, nullptr));
    dsa_config c{};
    c.batch = 1;
    c.heads = H;
    c.L = L;
    c.d = dk;
    c.k = 16;
    c.dtype = DSA_BF16;
    c.bits = 4;
    c.mask_mode = DSA_MASK_THRESHOLD;  // general CSR over every (head, row)
    c.scale = p.scale ? 1 : 0;
    c.frac_num = 1;
    c.frac_den = 1;
    c.cap = c.L;
    check(dsa_config_validate(&c));
    dsa_mask m{dc.as<uint32_t>(), drp.as<uint64_t>(), static_cast<int64_t>(cols.size()), nullptr};
    check(dsa_sparse_attention(&c, dq.get(), dkb.get(), dvb.get(), &m, dz.get(), nullptr));
    std::vector<uint16_t> hz(static_cast<size_t>(H * L * dv));
    check_cuda(cudaMemcpy(hz.data(), dz.get(), hz.size() * 2, cudaMemcpyDeviceToHost));
    Matrix out(static_cast<size_t>(L), static_cast<size_t>(H * dv), x.precision());
    for (int64_t h = 0; h < H; ++h)
        for (int64_t i = 0; i < L; ++i)
            for (int64_t j = 0; j < dv; ++j) {
                uint32_t u = static_cast<uint32_t>(hz[static_cast<size_t>((h * L + i) * dv + j)]) << 16;
                float f;
                std::memcpy(&f, &u, 4);
                out.raw()[static_cast<size_t>(i * H * dv + h * dv + j)] = f;
            }
    out.round_to_precision();
    return out;
}

}  // namespace dsattn::gpu
