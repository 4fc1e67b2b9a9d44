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

// ---------------------------------------------------------------- pipeline
// One (b,h) pair of the BASELINE path through reference functions
// (BASELINE.md 2): matmul(Q,P), matmul(K,P), quantize, exact-integer S~ via
// matmul_nt on the levels, mask selection, sddmm -> sparse_softmax -> spmm.
// mode: 0 row top-k, 1 colvec max-pool (v, keep), 2 block (bs, keep, diag),
//       3 causal threshold is not supported here (see oracle for O6).
struct RefPairArgs {
    const double *q, *k, *v, *p;
    int64_t L, d, kdim;
    int bits, f32, mode;
    int64_t keep, vec_v, block;
    int force_diag;
    double* z;
    uint32_t* mask_cols;  // may be null
};

static void run_pair(const RefPairArgs& a) {
    Matrix q = to_matrix(a.q, a.L, a.d, a.f32), k = to_matrix(a.k, a.L, a.d, a.f32);
    Matrix p = to_matrix(a.p, a.d, a.kdim, a.f32);
    double sq = 0, sk = 0;
    auto lq = levels_from_reference(matmul(q, p), a.bits, &sq);
    auto lk = levels_from_reference(matmul(k, p), a.bits, &sk);
    Matrix s = matmul_nt(int_matrix(lq, a.L, a.kdim), int_matrix(lk, a.L, a.kdim));
    SparseMask m(a.L);
    if (a.mode == 0) {
        m = predicted_topk_mask(s, a.keep);
    } else if (a.mode == 1) {
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
    } else {
        const int64_t nb = (a.L + a.block - 1) / a.block;
        for (int64_t ib = 0; ib < nb; ++ib) {
            Matrix bsum(1, nb);
            for (int64_t i = ib * a.block; i < std::min((ib + 1) * a.block, a.L); ++i)
                for (int64_t j = 0; j < a.L; ++j) bsum.raw()[j / a.block] += s(i, j);
            if (a.force_diag) bsum.raw()[ib] = 1e300;
            auto blocks = row_topk_indices(bsum, a.keep)[0];
            std::vector<uint32_t> cols;
            for (uint32_t jb : blocks)
                for (int64_t j = jb * a.block; j < std::min<int64_t>((jb + 1) * a.block, a.L); ++j)
                    cols.push_back(static_cast<uint32_t>(j));
            for (int64_t i = ib * a.block; i < std::min((ib + 1) * a.block, a.L); ++i) m.kept[i] = cols;
        }
    }
    SparseWeights w = sparse_softmax(sddmm(q, k, m, true));
    Matrix z = spmm(w, to_matrix(a.v, a.L, a.d, a.f32));
    std::memcpy(a.z, z.data(), z.size() * sizeof(double));
    if (a.mask_cols && (a.mode == 0)) {
        for (int64_t i = 0; i < a.L; ++i) std::memcpy(a.mask_cols + i * a.keep, m.kept[i].data(), a.keep * 4);
    }
}

// Runs `pairs` pairs over `threads` std::threads (contiguous chunks, as the
// reference's trainer splits batches, P/src/trainer.cpp:334-366).  Inputs are
// pair-major [pairs][L][d] doubles; p is [d][kdim].
int ref_pipeline(int64_t pairs, int threads, const double* q, const double* k, const double* v,
                 const double* p, int64_t L, int64_t d, int64_t kdim, int bits, int f32, int mode,
                 int64_t keep, int64_t vec_v, int64_t block, int force_diag, double* z) {
    return guarded([&] {
        const int T = std::max(1, std::min<int>(threads, static_cast<int>(pairs)));
        std::vector<std::thread> pool;
        std::vector<std::string> errs(T);
        for (int t = 0; t < T; ++t) {
            pool.emplace_back([&, t] {
                try {
                    for (int64_t pi = t; pi < pairs; pi += T) {
                        const size_t off = static_cast<size_t>(pi) * L * d;
                        run_pair(RefPairArgs{q + off, k + off, v + off, p, L, d, kdim, bits, f32,
                                             mode, keep, vec_v, block, force_diag, z + off,
                                             nullptr});
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
