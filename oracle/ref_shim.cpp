// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// library (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libdsattn_ref.so).  TEST INFRASTRUCTURE ONLY: used to pin the
// oracle restatement (tests/test_oracle_vs_reference.py), to generate golden
// vectors (oracle/gen_golden.py) and as the timed reference arm of bench.py.
//
// Every function composes reference entry points only (dsattn::matmul,
// quantize, row_topk_indices, predicted_topk_mask, colvec_mask,
// threshold_mask, sddmm, sparse_softmax, spmm, apply_additive_mask,
// row_softmax); the BASELINE extensions that have no reference function
// (max-pooled bands, block pooling, causal threshold) are built from those
// primitives exactly as SURVEY.md 8(c) O4-O6 prescribe.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "dsattn/attention.hpp"
#include "dsattn/dataflow.hpp"
#include "dsattn/kernels.hpp"
#include "dsattn/linalg.hpp"
#include "dsattn/maskgen.hpp"
#include "dsattn/predictor.hpp"
#include "dsattn/mask.hpp"
#include "dsattn/serialize.hpp"
#include "dsattn/sparse.hpp"

using namespace dsattn;

namespace {

thread_local std::string g_err;

Precision prec_of(int f32) { return f32 ? Precision::f32 : Precision::f64; }

Matrix to_matrix(const double* p, size_t r, size_t c, int f32) {
    Matrix m(r, c, prec_of(f32));
    std::memcpy(m.raw(), p, r * c * sizeof(double));
    m.round_to_precision();
    return m;
}

void from_matrix(const Matrix& m, double* out) {
    std::memcpy(out, m.data(), m.size() * sizeof(double));
}

SparseMask mask_from_csr(size_t L, const uint64_t* rowptr, const uint32_t* cols) {
    SparseMask m(L);
    for (size_t i = 0; i < L; ++i) m.kept[i].assign(cols + rowptr[i], cols + rowptr[i + 1]);
    return m;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 1;
    } catch (const ParamError& e) {
        g_err = e.what();
        return 2;
    } catch (const IoError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

// Integer levels recovered from the reference quantize() output: the
// reference returns level * s (predictor.cpp:43); s = max_abs(x) / qmax
// (predictor.cpp:38-41); lround(qt / s) recovers the level exactly.
std::vector<int32_t> levels_from_reference(const Matrix& x, int bits, double* s_out) {
    Matrix qt = quantize(x, QuantSpec{bits});
    const double qmax = static_cast<double>((1 << (bits - 1)) - 1);
    const double amax = max_abs(x);
    std::vector<int32_t> lv(x.size(), 0);
    *s_out = 0.0;
    if (amax == 0.0) return lv;
    const double s = amax / qmax;
    *s_out = s;
    for (size_t i = 0; i < x.size(); ++i) lv[i] = static_cast<int32_t>(std::lround(qt.data()[i] / s));
    return lv;
}

Matrix int_matrix(const std::vector<int32_t>& v, size_t r, size_t c) {
    Matrix m(r, c, Precision::f64);
    for (size_t i = 0; i < v.size(); ++i) m.raw()[i] = static_cast<double>(v[i]);
    return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
const char* ref_isa_name() { return kernels::isa_name(kernels::active_isa()); }

// matmul(Q, P) (P/src/linalg.cpp:11-17); f32 = both operands f32 Matrices.
int ref_project(const double* q, const double* p, int64_t L, int64_t d, int64_t k, int f32,
                double* x) {
    return guarded([&] { from_matrix(matmul(to_matrix(q, L, d, f32), to_matrix(p, d, k, f32)), x); });
}

// quantize(Matrix, QuantSpec) (P/src/predictor.cpp:34-45): dequantised output.
int ref_quantize(const double* x, int64_t rows, int64_t cols, int bits, int f32, double* y) {
    return guarded([&] { from_matrix(quantize(to_matrix(x, rows, cols, f32), QuantSpec{bits}), y); });
}

// Integer levels + scale through the reference quantize().
int ref_quantize_levels(const double* x, int64_t rows, int64_t cols, int bits, int f32,
                        int32_t* levels, double* scale) {
    return guarded([&] {
        auto lv = levels_from_reference(to_matrix(x, rows, cols, f32), bits, scale);
        std::memcpy(levels, lv.data(), lv.size() * sizeof(int32_t));
    });
}

// The reference predictor path (P/src/predictor.cpp:67-80) for one head and
// one side: r = matmul(x, p) when x != NULL (written to r_out), then
// levels / scale of quantize(matmul(r, w)).  f32: every Matrix is f32.
int ref_levels_wtilde(const double* x, const double* p, const double* r_in, const double* w, int64_t L,
                      int64_t dm, int64_t k, int bits, int f32, double* r_out, int32_t* levels, double* scale) {
    return guarded([&] {
        Matrix r = x ? matmul(to_matrix(x, L, dm, f32), to_matrix(p, dm, k, f32)) : to_matrix(r_in, L, k, f32);
        if (r_out) from_matrix(r, r_out);
        auto lv = levels_from_reference(matmul(r, to_matrix(w, k, k, f32)), bits, scale);
        std::memcpy(levels, lv.data(), lv.size() * sizeof(int32_t));
    });
}

// prediction_accuracy (P/src/maskgen.cpp:94-107) of two CSR masks.
int ref_prediction_accuracy(int64_t L, const uint64_t* rp_pred, const uint32_t* c_pred, const uint64_t* rp_orc,
                            const uint32_t* c_orc, double* out) {
    return guarded([&] {
        *out = prediction_accuracy(mask_from_csr(static_cast<size_t>(L), rp_pred, c_pred),
                                   mask_from_csr(static_cast<size_t>(L), rp_orc, c_orc));
    });
}

// dataflow::simulate (P/src/dataflow.cpp:48-62) on a CSR mask: total
// operand_fetches and pe_idle_steps for schedule kind (0 row_by_row,
// 1 row_parallel, 2 row_parallel_reordered) and band height.
int ref_dataflow_simulate(int64_t L, const uint64_t* rp, const uint32_t* cols, int kind, int64_t band,
                          uint64_t* fetches, uint64_t* idle) {
    return guarded([&] {
        const dataflow::ScheduleKind k = kind == 0 ? dataflow::ScheduleKind::row_by_row
                                         : kind == 1 ? dataflow::ScheduleKind::row_parallel
                                                     : dataflow::ScheduleKind::row_parallel_reordered;
        const dataflow::AccessTrace t =
            dataflow::simulate(mask_from_csr(static_cast<size_t>(L), rp, cols), {k, static_cast<size_t>(band)});
        *fetches = t.operand_fetches;
        *idle = t.pe_idle_steps;
    });
}

// init_projection (P/src/predictor.cpp:10-20): the reference's ternary P.
int ref_init_projection(int64_t d, int64_t k, uint64_t seed, double* p) {
    return guarded([&] { from_matrix(init_projection(static_cast<size_t>(d), static_cast<size_t>(k), seed).p, p); });
}

// row_topk_indices on a 1 x n row (P/src/linalg.cpp:69-85).
int ref_row_topk(const double* row, int64_t n, int64_t keep, uint32_t* out) {
    return guarded([&] {
        auto r = row_topk_indices(to_matrix(row, 1, n, 0), keep)[0];
        std::memcpy(out, r.data(), r.size() * sizeof(uint32_t));
    });
}

// predicted_topk_mask (P/src/maskgen.cpp:18-20) on a dense L x L score matrix.
int ref_topk_mask(const double* s, int64_t L, int64_t keep, uint32_t* cols) {
    return guarded([&] {
        SparseMask m = predicted_topk_mask(to_matrix(s, L, L, 0), keep);
        for (int64_t i = 0; i < L; ++i) std::memcpy(cols + i * keep, m.kept[i].data(), keep * 4);
    });
}

// colvec_mask as shipped (sum |s~| band score, P/src/maskgen.cpp:33-61).
int ref_colvec_mask(const double* s, int64_t L, int64_t v, int row_orient, double sparsity,
                    uint64_t* rowptr, uint32_t* cols) {
    return guarded([&] {
        SparseMask m = colvec_mask(to_matrix(s, L, L, 0),
                                   ColVecSpec{static_cast<size_t>(v),
                                              row_orient ? VecOrientation::row : VecOrientation::col},
                                   sparsity);
        rowptr[0] = 0;
        for (int64_t i = 0; i < L; ++i) {
            rowptr[i + 1] = rowptr[i] + m.kept[i].size();
            if (cols) std::memcpy(cols + rowptr[i], m.kept[i].data(), m.kept[i].size() * 4);
        }
    });
}

// threshold_mask as shipped (P/src/maskgen.cpp:22-31).
int ref_threshold_mask(const double* s, int64_t L, double theta, int post_softmax,
                       uint64_t* rowptr, uint32_t* cols) {
    return guarded([&] {
        SparseMask m = threshold_mask(to_matrix(s, L, L, 0), theta, post_softmax != 0);
        rowptr[0] = 0;
        for (int64_t i = 0; i < L; ++i) {
            rowptr[i + 1] = rowptr[i] + m.kept[i].size();
            if (cols) std::memcpy(cols + rowptr[i], m.kept[i].data(), m.kept[i].size() * 4);
        }
    });
}

// O4 from reference primitives: band score = max over the band rows of the
// integer score, then row_topk_indices on the 1 x L pooled row.
int ref_colvec_maxpool_mask(const double* s_int, int64_t L, int64_t v, int64_t keep,
                            uint32_t* band_cols) {
    return guarded([&] {
        const int64_t nb = (L + v - 1) / v;
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t r0 = b * v, r1 = std::min(r0 + v, L);
            Matrix pooled(1, L);
            for (int64_t j = 0; j < L; ++j) {
                double m = s_int[r0 * L + j];
                for (int64_t i = r0 + 1; i < r1; ++i) m = std::max(m, s_int[i * L + j]);
                pooled.raw()[j] = m;
            }
            auto cols = row_topk_indices(pooled, keep)[0];
            std::memcpy(band_cols + b * keep, cols.data(), keep * 4);
        }
    });
}

// sddmm -> sparse_softmax -> spmm for one head (P/src/sparse.cpp:38-91).
int ref_sparse_attention(const double* q, const double* k, const double* v, int64_t L,
                         int64_t d, int64_t dv, int f32, const uint64_t* rowptr,
                         const uint32_t* cols, int scale, double* z, uint8_t* empty_row,
                         uint64_t* counters /* sddmm_mults, spmm_mults, softmax_exps */) {
    return guarded([&] {
        SparseMask m = mask_from_csr(L, rowptr, cols);
        op_counters().reset();
        SparseWeights w = sparse_softmax(sddmm(to_matrix(q, L, d, f32), to_matrix(k, L, d, f32), m,
                                               scale != 0));
        Matrix out = spmm(w, to_matrix(v, L, dv, f32));
        from_matrix(out, z);
        if (empty_row) std::memcpy(empty_row, w.empty_row.data(), L);
        if (counters) {
            counters[0] = op_counters().sddmm_mults;
            counters[1] = op_counters().spmm_mults;
            counters[2] = op_counters().softmax_exps;
        }
    });
}

// Dense Eq. 4 with the additive mask (P/src/attention.cpp:48-71) per head.
int ref_masked_attention(const double* q, const double* k, const double* v, int64_t L,
                         int64_t d, int64_t dv, const uint64_t* rowptr, const uint32_t* cols,
                         int scale, double* z) {
    return guarded([&] {
        SparseMask m = mask_from_csr(L, rowptr, cols);
        Matrix s = attention_scores(to_matrix(q, L, d, 0), to_matrix(k, L, d, 0), scale != 0);
        Matrix a = row_softmax(apply_additive_mask(s, m));
        from_matrix(matmul(a, to_matrix(v, L, dv, 0)), z);
    });
}

}  // extern "C"

// ------------------------------------------- block and causal threshold (O5, O6)
// Exact-integer S~ rows [r0, r1) through the reference matmul_nt
// (P/src/linalg.cpp:19-27) on integer-valued f64 level Matrices.
static Matrix score_rows(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k, int64_t r0, int64_t r1) {
    Matrix a(static_cast<size_t>(r1 - r0), static_cast<size_t>(k), Precision::f64);
    for (int64_t i = 0; i < (r1 - r0) * k; ++i) a.raw()[i] = static_cast<double>(lq[r0 * k + i]);
    Matrix b(static_cast<size_t>(L), static_cast<size_t>(k), Precision::f64);
    for (int64_t i = 0; i < L * k; ++i) b.raw()[i] = static_cast<double>(lk[i]);
    return matmul_nt(a, b);
}

// O5 from reference primitives: per block row, the mean of S~ over each
// bs x bs block (sum / count, both exact integers in f64), the diagonal
// block forced first (+1e300), then row_topk_indices (P/src/linalg.cpp:69-85,
// ties to the lowest block) on the 1 x nb row of means.
static std::vector<std::vector<uint32_t>> block_lists(const int32_t* lq, const int32_t* lk, int64_t L,
                                                      int64_t k, int64_t bs, int64_t keep, int force_diag) {
    const int64_t nb = (L + bs - 1) / bs;
    std::vector<std::vector<uint32_t>> out(static_cast<size_t>(nb));
    for (int64_t ib = 0; ib < nb; ++ib) {
        const int64_t r0 = ib * bs, r1 = std::min(r0 + bs, L);
        const Matrix s = score_rows(lq, lk, L, k, r0, r1);
        Matrix mean(1, static_cast<size_t>(nb), Precision::f64);
        for (int64_t jb = 0; jb < nb; ++jb) {
            const int64_t c0 = jb * bs, c1 = std::min(c0 + bs, L);
            double sum = 0.0;
            for (int64_t i = 0; i < r1 - r0; ++i)
                for (int64_t j = c0; j < c1; ++j) sum += s(static_cast<size_t>(i), static_cast<size_t>(j));
            mean.raw()[jb] = sum / static_cast<double>((r1 - r0) * (c1 - c0));
        }
        if (force_diag) mean.raw()[ib] = 1e300;
        out[static_cast<size_t>(ib)] = row_topk_indices(mean, static_cast<size_t>(keep))[0];
    }
    return out;
}

// O6 from reference primitives, one query row: p = row_softmax(c * S~)
// (P/src/linalg.cpp:51-67) over the candidates j <= i (causal) or all j,
// kept where p >= theta (the threshold_mask rule, P/src/maskgen.cpp:29);
// more than `cap` survivors -> the cap largest by S~ via row_topk_indices
// (ties to the lowest index).
static std::vector<uint32_t> threshold_row(const Matrix& s, size_t ri, int64_t i, int64_t L, double c,
                                           double theta, int64_t cap, int causal, double* probs) {
    const int64_t n = causal ? i + 1 : L;
    Matrix x(1, static_cast<size_t>(n), Precision::f64);
    for (int64_t j = 0; j < n; ++j) x.raw()[j] = s(ri, static_cast<size_t>(j));
    const Matrix p = row_softmax(scale(x, c));
    if (probs) std::memcpy(probs, p.data(), static_cast<size_t>(n) * sizeof(double));
    std::vector<uint32_t> kept;
    for (int64_t j = 0; j < n; ++j)
        if (p(0, static_cast<size_t>(j)) >= theta) kept.push_back(static_cast<uint32_t>(j));
    if (static_cast<int64_t>(kept.size()) > cap) {
        Matrix key(1, static_cast<size_t>(n), Precision::f64);
        for (int64_t j = 0; j < n; ++j) key.raw()[j] = -1e300;
        for (uint32_t j : kept) key.raw()[j] = x(0, j);
        kept = row_topk_indices(key, static_cast<size_t>(cap))[0];
    }
    return kept;
}

static void threshold_lists(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k, double c, double theta,
                            int64_t cap, int causal, std::vector<std::vector<uint32_t>>& rows) {
    rows.assign(static_cast<size_t>(L), {});
    constexpr int64_t kChunk = 256;  // S~ rows materialised at a time
    for (int64_t r0 = 0; r0 < L; r0 += kChunk) {
        const int64_t r1 = std::min(r0 + kChunk, L);
        const Matrix s = score_rows(lq, lk, L, k, r0, r1);
        for (int64_t i = r0; i < r1; ++i)
            rows[static_cast<size_t>(i)] = threshold_row(s, static_cast<size_t>(i - r0), i, L, c, theta, cap, causal, nullptr);
    }
}

extern "C" {

// Block-column lists [ceil(L/bs)][keep] of the BLOCK mode.
int ref_block_mask(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k, int64_t bs, int64_t keep,
                   int force_diag, uint32_t* block_cols) {
    return guarded([&] {
        const auto lists = block_lists(lq, lk, L, k, bs, keep, force_diag);
        for (size_t b = 0; b < lists.size(); ++b)
            std::memcpy(block_cols + b * keep, lists[b].data(), static_cast<size_t>(keep) * 4);
    });
}

// Causal (or full-row) softmax threshold + cap as CSR; cols == NULL: rowptr only.
int ref_causal_threshold_mask(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k, double c,
                              double theta, int64_t cap, int causal, uint64_t* rowptr, uint32_t* cols) {
    return guarded([&] {
        std::vector<std::vector<uint32_t>> rows;
        threshold_lists(lq, lk, L, k, c, theta, cap, causal, rows);
        rowptr[0] = 0;
        for (int64_t i = 0; i < L; ++i) {
            rowptr[i + 1] = rowptr[i] + rows[i].size();
            if (cols) std::memcpy(cols + rowptr[i], rows[i].data(), rows[i].size() * 4);
        }
    });
}

// The reference softmax probabilities of query row i (n = i+1 causal, else L
// values) -- to show that any disagreement with the oracle lies at theta.
int ref_threshold_row_probs(const int32_t* lq, const int32_t* lk, int64_t L, int64_t k, double c, int64_t i,
                            int causal, double* probs) {
    return guarded([&] {
        const Matrix s = score_rows(lq, lk, L, k, i, i + 1);
        threshold_row(s, 0, i, L, c, 0.0, L + 1, causal, probs);
    });
}

// Seeded BASELINE inputs drawn with the reference Rng
// (P/include/dsattn/rng.hpp:14-78): per pair the substream split(1000 + pair)
// of Rng(seed); Q/K/V ~ normal(), planted keys by partial Fisher-Yates with
// uniform_int, +3u / +0.5u (u from split(0)), optional local band windows,
// P = normal() / sqrt(k) from split(1).  Values are returned as doubles
// rounded to the dtype (bf16 round-to-nearest-even through float, or f32).
int ref_generate(int64_t L, int64_t d, int64_t kdim, int bf16, uint64_t seed, int planted_pm, int band_w,
                 int64_t pair0, int64_t npairs, double* q, double* k, double* v, double* p) {
    return guarded([&] {
        auto round_to = [&](double x) {
            float f = static_cast<float>(x);
            if (!bf16) return static_cast<double>(f);
            uint32_t u;
            std::memcpy(&u, &f, 4);
            if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<double>(f);
            u += 0x7fffu + ((u >> 16) & 1u);
            u &= 0xffff0000u;
            std::memcpy(&f, &u, 4);
            return static_cast<double>(f);
        };
        auto unit = [&](Rng& g) {
            std::vector<double> u(static_cast<size_t>(d));
            double n2 = 0.0;
            for (auto& x : u) {
                x = g.normal();
                n2 += x * x;
            }
            const double inv = 1.0 / std::sqrt(n2);
            for (auto& x : u) x *= inv;
            return u;
        };
        Rng r0(seed);
        Rng shared = r0.split(0);
        const std::vector<double> u = unit(shared);
        if (p) {
            Rng r1(seed);
            Rng gp = r1.split(1);
            const double sd = 1.0 / std::sqrt(static_cast<double>(kdim));
            for (int64_t i = 0; i < d * kdim; ++i) p[i] = static_cast<double>(static_cast<float>(sd * gp.normal()));
        }
        for (int64_t pi = 0; pi < npairs; ++pi) {
            Rng root(seed);
            Rng g = root.split(1000 + static_cast<uint64_t>(pair0 + pi));
            std::vector<double> Q(L * d), K(L * d), V(L * d);
            for (auto& x : Q) x = g.normal();
            for (auto& x : K) x = g.normal();
            for (auto& x : V) x = g.normal();
            const int64_t npl = (static_cast<int64_t>(planted_pm) * L + 500) / 1000;
            std::vector<int64_t> pool(L);
            for (int64_t j = 0; j < L; ++j) pool[j] = j;
            for (int64_t t = 0; t < npl; ++t) {
                const int64_t r = t + static_cast<int64_t>(g.uniform_int(static_cast<uint64_t>(L - t)));
                std::swap(pool[t], pool[r]);
                for (int64_t c2 = 0; c2 < d; ++c2) K[pool[t] * d + c2] += 3.0 * u[c2];
            }
            for (int64_t i = 0; i < L; ++i)
                for (int64_t c2 = 0; c2 < d; ++c2) Q[i * d + c2] += 0.5 * u[c2];
            if (band_w > 0) {
                const int64_t nw = (L + band_w - 1) / band_w;
                for (int64_t w = 0; w < nw; ++w) {
                    const std::vector<double> e = unit(g);
                    for (int64_t i = w * band_w; i < std::min<int64_t>(L, (w + 1) * band_w); ++i)
                        for (int64_t c2 = 0; c2 < d; ++c2) {
                            Q[i * d + c2] += e[c2];
                            K[i * d + c2] += e[c2];
                        }
                }
            }
            const size_t off = static_cast<size_t>(pi) * L * d;
            for (int64_t i = 0; i < L * d; ++i) {
                q[off + i] = round_to(Q[i]);
                k[off + i] = round_to(K[i]);
                v[off + i] = round_to(V[i]);
            }
        }
    });
}

}  // extern "C"

extern "C" {

// ---------------------------------------------------------------- pipeline
// One (b,h) pair of the BASELINE path through reference functions
// (BASELINE.md 2): matmul(Q,P), matmul(K,P), quantize, exact-integer S~ via
// matmul_nt on the levels, mask selection, sddmm -> sparse_softmax -> spmm.
// mode: 0 row top-k (per_row: quantize() applied to each 1 x k row, ranked
//       by S~ * s_k[j] -- SURVEY S5), 1 colvec max-pool (v, keep), 2 block
//       (bs, keep, diag; O5), 3 softmax threshold + cap, causal (O6).
struct RefPairArgs {
    const double *q, *k, *v, *p;
    int64_t L, d, kdim;
    int bits, f32, mode, per_row;
    int64_t keep, vec_v, block;
    int force_diag;
    int64_t frac_num, frac_den, cap;
    int causal;
    double* z;
};

static std::vector<int32_t> row_levels(const Matrix& x, int bits, std::vector<double>& s) {
    std::vector<int32_t> lv(x.size());
    s.assign(x.rows(), 0.0);
    for (size_t i = 0; i < x.rows(); ++i) {
        Matrix r(1, x.cols(), Precision::f64);
        std::memcpy(r.raw(), x.data() + i * x.cols(), x.cols() * sizeof(double));
        auto l = levels_from_reference(r, bits, &s[i]);
        std::memcpy(lv.data() + i * x.cols(), l.data(), l.size() * sizeof(int32_t));
    }
    return lv;
}

static void run_pair(const RefPairArgs& a) {
    Matrix q = to_matrix(a.q, a.L, a.d, a.f32), k = to_matrix(a.k, a.L, a.d, a.f32);
    Matrix p = to_matrix(a.p, a.d, a.kdim, a.f32);
    double sq = 0, sk = 0;
    std::vector<double> skr;
    std::vector<int32_t> lq, lk;
    if (a.per_row) {
        std::vector<double> sqr;
        lq = row_levels(matmul(q, p), a.bits, sqr);
        lk = row_levels(matmul(k, p), a.bits, skr);
    } else {
        lq = levels_from_reference(matmul(q, p), a.bits, &sq);
        lk = levels_from_reference(matmul(k, p), a.bits, &sk);
    }
    SparseMask m(a.L);
    if (a.mode == 3) {
        const double c = sq * sk / std::sqrt(static_cast<double>(a.d));
        const double theta = static_cast<double>(a.frac_den) / (static_cast<double>(a.frac_num) * a.L);
        threshold_lists(lq.data(), lk.data(), a.L, a.kdim, c, theta, a.cap, a.causal, m.kept);
    } else if (a.mode == 2) {
        const auto lists = block_lists(lq.data(), lk.data(), a.L, a.kdim, a.block, a.keep, a.force_diag);
        for (int64_t ib = 0; ib < static_cast<int64_t>(lists.size()); ++ib) {
            std::vector<uint32_t> cols;
            for (uint32_t jb : lists[ib])
                for (int64_t j = jb * a.block; j < std::min<int64_t>((jb + 1) * a.block, a.L); ++j)
                    cols.push_back(static_cast<uint32_t>(j));
            for (int64_t i = ib * a.block; i < std::min((ib + 1) * a.block, a.L); ++i) m.kept[i] = cols;
        }
    } else {
        Matrix s = matmul_nt(int_matrix(lq, a.L, a.kdim), int_matrix(lk, a.L, a.kdim));
        if (a.mode == 0) {
            if (a.per_row)
                for (int64_t i = 0; i < a.L; ++i)
                    for (int64_t j = 0; j < a.L; ++j) s.raw()[i * a.L + j] *= skr[j];
            m = predicted_topk_mask(s, a.keep);
        } else {
            for (int64_t b0 = 0; b0 < a.L; b0 += a.vec_v) {
                const int64_t b1 = std::min(b0 + a.vec_v, a.L);
                Matrix pooled(1, a.L);
                for (int64_t j = 0; j < a.L; ++j) {
                    double mx = s(b0, j);
                    for (int64_t i = b0 + 1; i < b1; ++i) mx = std::max(mx, s(i, j));
                    pooled.raw()[j] = mx;
                }
                auto cols = row_topk_indices(pooled, a.keep)[0];
                for (int64_t i = b0; i < b1; ++i) m.kept[i] = cols;
            }
        }
    }
    SparseWeights w = sparse_softmax(sddmm(q, k, m, true));
    Matrix z = spmm(w, to_matrix(a.v, a.L, a.d, a.f32));
    std::memcpy(a.z, z.data(), z.size() * sizeof(double));
}

// Runs `pairs` pairs over `threads` std::threads (pairs strided over the
// threads, as the reference's trainer splits batches over a thread pool,
// P/src/trainer.cpp:334-366).  Inputs are pair-major [pairs][L][d] doubles;
// p is [d][kdim].
int ref_pipeline(int64_t pairs, int threads, const double* q, const double* k, const double* v,
                 const double* p, int64_t L, int64_t d, int64_t kdim, int bits, int f32, int mode,
                 int per_row, int64_t keep, int64_t vec_v, int64_t block, int force_diag, int64_t frac_num,
                 int64_t frac_den, int64_t cap, int causal, double* z) {
    return guarded([&] {
        const int T = std::max(1, std::min<int>(threads, static_cast<int>(pairs)));
        std::vector<std::thread> pool;
        std::vector<std::string> errs(T);
        for (int t = 0; t < T; ++t) {
            pool.emplace_back([&, t] {
                try {
                    for (int64_t pi = t; pi < pairs; pi += T) {
                        const size_t off = static_cast<size_t>(pi) * L * d;
                        run_pair(RefPairArgs{q + off, k + off, v + off, p, L, d, kdim, bits, f32, mode, per_row,
                                             keep, vec_v, block, force_diag, frac_num, frac_den, cap, causal,
                                             z + off});
                    }
                } catch (const std::exception& e) {
                    errs[t] = e.what();
                }
            });
        }
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (!e.empty()) throw ParamError(e);
    });
}

// ---- fixture / wire formats (P/src/mask.cpp:75-114, P/src/sparse.cpp:122-171,
// P/src/serialize.cpp:38-95): the reference's own writers and readers, so
// the GPU harness's files are pinned against them.
int ref_write_mask(const char* path, int64_t L, const uint64_t* rowptr, const uint32_t* cols) {
    return guarded([&] { write_mask(path, mask_from_csr(static_cast<size_t>(L), rowptr, cols)); });
}

// Two calls: cols == NULL returns L (*l_out) and nnz (*nnz_out); then fills
// rowptr[L+1] and cols[nnz].
int ref_read_mask(const char* path, int64_t* l_out, int64_t* nnz_out, uint64_t* rowptr, uint32_t* cols) {
    return guarded([&] {
        const SparseMask m = read_mask(path);
        *l_out = static_cast<int64_t>(m.l);
        *nnz_out = static_cast<int64_t>(m.nnz());
        if (!cols) return;
        uint64_t off = 0;
        rowptr[0] = 0;
        for (size_t i = 0; i < m.l; ++i) {
            for (uint32_t c : m.kept[i]) cols[off++] = c;
            rowptr[i + 1] = off;
        }
    });
}

int ref_write_sparse_scores(const char* path, int64_t L, const uint64_t* rowptr, const uint32_t* cols,
                            const double* values) {
    return guarded([&] {
        SparseScores s;
        s.mask = mask_from_csr(static_cast<size_t>(L), rowptr, cols);
        s.row_offsets.assign(rowptr, rowptr + L + 1);
        s.values.assign(values, values + rowptr[L]);
        write_sparse_scores(path, s);
    });
}

int ref_read_sparse_scores(const char* path, int64_t* l_out, int64_t* nnz_out, uint64_t* rowptr,
                           uint32_t* cols, double* values) {
    return guarded([&] {
        const SparseScores s = read_sparse_scores(path);
        *l_out = static_cast<int64_t>(s.mask.l);
        *nnz_out = static_cast<int64_t>(s.values.size());
        if (!cols) return;
        uint64_t off = 0;
        rowptr[0] = 0;
        for (size_t i = 0; i < s.mask.l; ++i) {
            for (uint32_t c : s.mask.kept[i]) cols[off++] = c;
            rowptr[i + 1] = off;
        }
        std::memcpy(values, s.values.data(), s.values.size() * sizeof(double));
    });
}

// One-entry DSAC container (data: rows*cols doubles, rounded to f32 when
// f32 != 0, as the reference stores f32 Matrices).
int ref_write_container1(const char* path, const char* name, int64_t rows, int64_t cols, int f32,
                         const double* data, const char* meta) {
    return guarded([&] {
        write_container(path, {{name, to_matrix(data, static_cast<size_t>(rows), static_cast<size_t>(cols), f32)}},
                        meta ? meta : "");
    });
}

// Entry `name`: first call (out == NULL) reports rows, cols, precision and
// the meta length; the second copies the data (as doubles) and the meta.
int ref_read_container1(const char* path, const char* name, int64_t* rows, int64_t* cols, int* f32,
                        double* out, int64_t* meta_len, char* meta) {
    return guarded([&] {
        const Container c = read_container(path);
        const Matrix& m = c.find(name);
        *rows = static_cast<int64_t>(m.rows());
        *cols = static_cast<int64_t>(m.cols());
        *f32 = m.precision() == Precision::f32 ? 1 : 0;
        *meta_len = static_cast<int64_t>(c.meta.size());
        if (out) from_matrix(m, out);
        if (meta) std::memcpy(meta, c.meta.data(), c.meta.size());
    });
}

}  // extern "C"
