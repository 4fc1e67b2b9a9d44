// C++ drop-in checks: include/dsattn_gpu.hpp used exactly as a reference
// caller would (reference types, value semantics, reference exceptions),
// compared with the reference implementation linked into the same binary.
// Built by oracle/Makefile (target shim_test) into oracle/_ref/test_shim;
// run on a GPU by tests/test_gpu_cpp_shim.py.  Cases mirror the reference's
// own tests (P/tests/test_linalg.cpp:97-101, test_maskgen.cpp, test_sparse.cpp).
#include <algorithm>
#include <cmath>
#include <memory>
#include <cstring>
#include <cstdio>
#include <vector>

#include "dsattn/attention.hpp"
#include "dsattn/kernels.hpp"
#include "dsattn/linalg.hpp"
#include "dsattn/maskgen.hpp"
#include "dsattn/predictor.hpp"
#include "dsattn/sparse.hpp"
#include "dsattn_gpu.hpp"

using namespace dsattn;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (cond) {                                                        \
            ++g_pass;                                                      \
        } else {                                                           \
            ++g_fail;                                                      \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);   \
        }                                                                  \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static Matrix bf16_normal(size_t r, size_t c, Rng& rng) {
    Matrix m(r, c);
    for (size_t i = 0; i < m.size(); ++i) {
        float f = static_cast<float>(rng.normal());
        uint32_t u;
        std::memcpy(&u, &f, 4);
        u &= 0xffff0000u;
        std::memcpy(&f, &u, 4);
        m.raw()[i] = f;
    }
    return m;
}

// Integer levels via the reference: quantize(matmul(X, P)) / s
static Matrix ref_levels(const Matrix& x, const Matrix& p, int bits) {
    Matrix xp = matmul(x, p);
    Matrix qt = quantize(xp, QuantSpec{bits});
    const double s = max_abs(xp) / ((1 << (bits - 1)) - 1);
    Matrix lv(qt.rows(), qt.cols());
    for (size_t i = 0; i < qt.size(); ++i) lv.raw()[i] = s == 0 ? 0 : std::lround(qt.data()[i] / s);
    return lv;
}

#define STEP(name) std::printf("-- %s\n", name)

int main() {
    std::setvbuf(stdout, nullptr, _IONBF, 0);
    Rng rng(2110);
    const size_t L = 300, d = 64, k = 16;
    Matrix q = bf16_normal(L, d, rng), kk = bf16_normal(L, d, rng), v = bf16_normal(L, d, rng);
    Matrix p = random_normal(d, k, 0.0, 0.25, rng, Precision::f32).as_precision(Precision::f64);

    // levels == the reference's quantize (bit-exact)
    gpu::Levels lv = gpu::predict(q, kk, p, QuantSpec{4});
    Matrix rq = ref_levels(q, p, 4), rk = ref_levels(kk, p, 4);
    CHECK(max_abs_diff(lv.q, rq) == 0.0);
    CHECK(max_abs_diff(lv.k, rk) == 0.0);

    // predicted_topk_mask == reference predicted_topk_mask on exact S~
    SparseMask g = gpu::predicted_topk_mask(q, kk, p, QuantSpec{4}, 17);
    SparseMask r = predicted_topk_mask(matmul_nt(rq, rk), 17);
    CHECK(g == r);

    // colvec (max-pooled) == reference primitives composition
    SparseMask gc = gpu::colvec_mask(q, kk, p, QuantSpec{4}, ColVecSpec{8, VecOrientation::col}, 9);
    {
        Matrix s = matmul_nt(rq, rk);
        bool ok = true;
        for (size_t b0 = 0; b0 < L; b0 += 8) {
            Matrix pooled(1, L);
            for (size_t j = 0; j < L; ++j) {
                double m = s(b0, j);
                for (size_t i = b0 + 1; i < std::min(L, b0 + 8); ++i) m = std::max(m, s(i, j));
                pooled.raw()[j] = m;
            }
            auto cols = row_topk_indices(pooled, 9)[0];
            for (size_t i = b0; i < std::min(L, b0 + 8); ++i) ok &= gc.kept[i] == cols;
        }
        CHECK(ok);
    }

    // tie known answer: S row [1, 7, 4, 7] -> top-2 {1, 3} (P/tests/test_linalg.cpp:97-101)
    {
        Matrix q1(4, 16), k1(4, 16), eye(16, 16, Precision::f32);
        for (size_t i = 0; i < 16; ++i) eye.set(i, i, 1.0);
        for (size_t i = 0; i < 4; ++i) q1.set(i, 0, 1.0);
        const double col0[4] = {1.0, 9.0, 5.0, 9.0};
        for (size_t i = 0; i < 4; ++i) k1.set(i, 0, col0[i]);
        SparseMask t = gpu::predicted_topk_mask(q1, k1, eye.as_precision(Precision::f64), QuantSpec{4}, 2);
        CHECK((t.kept[0] == std::vector<uint32_t>{1, 3}));
    }

    // sparse attention vs the reference sddmm -> sparse_softmax -> spmm
    {
        Matrix qf = q.as_precision(Precision::f32), kf = kk.as_precision(Precision::f32),
               vf = v.as_precision(Precision::f32);
        Matrix zg = gpu::sparse_attention(qf, kf, vf, r, true);
        Matrix zr = spmm(sparse_softmax(sddmm(qf, kf, r, true)), vf);
        CHECK(max_abs_diff(zg, zr) <= 1e-5 * std::max(1.0, max_abs(zr)));
        // empty row -> zero, flagged (P/tests/test_sparse.cpp:89-97)
        SparseMask e = r;
        e.kept[3].clear();
        std::vector<uint8_t> flags;
        Matrix ze = gpu::sparse_attention(qf, kf, vf, e, true, &flags);
        bool zero = true;
        for (size_t j = 0; j < d; ++j) zero &= ze(3, j) == 0.0;
        CHECK(zero && flags[3] == 1 && flags[2] == 0);
    }

    STEP("project_qkv");
    // project_qkv vs the reference (P/src/attention.cpp:36-46) on bf16-exact
    // operands: within the bf16 bar per head
    {
        Rng prng(99);
        const size_t dm = 128, Lx = 200, H = 3;
        AttentionParams ap = random_attention_params(dm, 64, 64, H, prng);
        auto to_bf16 = [](Matrix& m) {
            for (size_t i = 0; i < m.size(); ++i) {
                float f = static_cast<float>(m.data()[i]);
                uint32_t u;
                std::memcpy(&u, &f, 4);
                u &= 0xffff0000u;
                std::memcpy(&f, &u, 4);
                m.raw()[i] = f;
            }
        };
        for (auto* ws : {&ap.wq, &ap.wk, &ap.wv})
            for (Matrix& w : *ws) to_bf16(w);
        Matrix x = random_normal(Lx, dm, 0.0, 1.0, prng);
        to_bf16(x);
        Qkv g = gpu::project_qkv(x, ap), ref = project_qkv(x, ap);
        for (size_t h = 0; h < H; ++h) {
            CHECK(max_abs_diff(g.q[h], ref.q[h]) <= 1e-2 * max_abs(ref.q[h]));
            CHECK(max_abs_diff(g.k[h], ref.k[h]) <= 1e-2 * max_abs(ref.k[h]));
            CHECK(max_abs_diff(g.v[h], ref.v[h]) <= 1e-2 * max_abs(ref.v[h]));
        }
        CHECK(throws<ShapeError>([&] { gpu::project_qkv(Matrix(Lx, dm + 1), ap); }));
        // the layer-level sparse_attention (P/src/sparse.cpp:93-120) with one
        // predicted mask per head: Q/K/V and Z pass through bf16 (two
        // roundings), bar 2e-2 of max |Z|
        std::vector<SparseMask> masks;
        for (size_t h = 0; h < H; ++h)
            masks.push_back(predicted_topk_mask(matmul_nt(ref.q[h], ref.k[h]), 20 + 5 * h));
        masks[1].kept[7].clear();  // an empty row: zero output
        Matrix zg = gpu::sparse_attention(x, ap, std::span<const SparseMask>(masks));
        Matrix zr = sparse_attention(x, ap, std::span<const SparseMask>(masks));
        CHECK(zg.rows() == zr.rows() && zg.cols() == zr.cols());
        CHECK(max_abs_diff(zg, zr) <= 2e-2 * max_abs(zr));
        CHECK(zg(7, 64) == 0.0 && zg(7, 127) == 0.0);
        CHECK(throws<ShapeError>([&] { gpu::sparse_attention(x, ap, std::span<const SparseMask>(masks.data(), 2)); }));
    }

    STEP("threshold");
    // threshold_mask mirror.  Full rows, no cap: the reference threshold_mask
    // itself on c * S~ post-softmax (P/src/maskgen.cpp:22-31).  Causal + cap:
    // row_softmax over j <= i, ">= theta", the cap largest S~ by
    // row_topk_indices.
    {
        const double sq = max_abs(matmul(q, p)) / 7.0, sk = max_abs(matmul(kk, p)) / 7.0;
        const double c = sq * sk / std::sqrt(static_cast<double>(d));
        const Matrix s = matmul_nt(rq, rk);
        SparseMask gt = gpu::threshold_mask(q, kk, p, QuantSpec{4}, 1, 20, L, false);
        CHECK(gt == threshold_mask(scale(s, c), 20.0 / L, true));
        const double theta = 4.0 / L;
        SparseMask gcz = gpu::threshold_mask(q, kk, p, QuantSpec{4}, 1, 4, 6, true);
        bool ok = true;
        size_t capped = 0;
        for (size_t i = 0; i < L; ++i) {
            Matrix x(1, i + 1);
            for (size_t j = 0; j <= i; ++j) x.raw()[j] = s(i, j);
            const Matrix pr = row_softmax(scale(x, c));
            std::vector<uint32_t> kept;
            for (uint32_t j = 0; j <= i; ++j)
                if (pr(0, j) >= theta) kept.push_back(j);
            if (kept.size() > 6) {
                ++capped;
                Matrix key(1, i + 1);
                for (size_t j = 0; j <= i; ++j) key.raw()[j] = -1e300;
                for (uint32_t j : kept) key.raw()[j] = x(0, j);
                kept = row_topk_indices(key, 6)[0];
            }
            ok &= gcz.kept[i] == kept;
        }
        CHECK(ok);
        CHECK(capped > 0);
    }

    STEP("block");
    // block_mask mirror: 32 x 32 block means, the diagonal block
    // forced, row_topk_indices over the block row; L = 300 leaves a ragged
    // 12-row / 12-column last block
    {
        const Matrix s = matmul_nt(rq, rk);
        const size_t bs = 32, nb = (L + bs - 1) / bs, keep = 3;
        SparseMask gb = gpu::block_mask(q, kk, p, QuantSpec{4}, bs, keep, true);
        bool ok = true;
        for (size_t ib = 0; ib < nb; ++ib) {
            Matrix mean(1, nb);
            const size_t r0 = ib * bs, r1 = std::min(L, r0 + bs);
            for (size_t jb = 0; jb < nb; ++jb) {
                const size_t c0 = jb * bs, c1 = std::min(L, c0 + bs);
                double sum = 0;
                for (size_t i = r0; i < r1; ++i)
                    for (size_t j = c0; j < c1; ++j) sum += s(i, j);
                mean.raw()[jb] = sum / static_cast<double>((r1 - r0) * (c1 - c0));
            }
            mean.raw()[ib] = 1e300;
            std::vector<uint32_t> cols;
            const std::vector<uint32_t> top = row_topk_indices(mean, keep)[0];
            for (uint32_t jb : top)
                for (size_t j = jb * bs; j < std::min(L, (jb + 1) * bs); ++j) cols.push_back(static_cast<uint32_t>(j));
            for (size_t i = r0; i < r1; ++i) ok &= gb.kept[i] == cols;
        }
        CHECK(ok);
    }

    STEP("wtilde");
    // the reference predictor with its per-head W~: approx_scores(x, pp)
    // levels bit-exact (R = X P, quantize(R W~)), and the caller's
    // predicted_topk_mask on the exact integer S~ (P/src/trainer.cpp:162-195)
    {
        Rng wrng(7);
        const size_t dm = 96, Lx = 257;
        auto proj = std::make_shared<const ProjectionMatrix>(init_projection(dm, k, 11));
        PredictorParams pp = random_predictor_params(proj, 0.3, wrng, QuantSpec{4});
        Matrix x = random_normal(Lx, dm, 0.0, 1.0, wrng);
        const Matrix r = matmul(x, proj->p);
        auto lev = [&](const Matrix& w) {
            const Matrix xw = matmul(r, w);
            const Matrix qt = quantize(xw, QuantSpec{4});
            const double sc = max_abs(xw) / 7.0;
            Matrix lv(qt.rows(), qt.cols());
            for (size_t i = 0; i < qt.size(); ++i) lv.raw()[i] = std::lround(qt.data()[i] / sc);
            return lv;
        };
        const Matrix lq = lev(pp.wq), lk = lev(pp.wk);
        gpu::Levels gl = gpu::approx_levels(x, pp);
        CHECK(max_abs_diff(gl.q, lq) == 0.0 && max_abs_diff(gl.k, lk) == 0.0);
        CHECK(gl.scale_q[0] == max_abs(matmul(r, pp.wq)) / 7.0);
        CHECK(gpu::predicted_topk_mask(x, pp, 17) == predicted_topk_mask(matmul_nt(lq, lk), 17));
        CHECK(gpu::predicted_topk_mask_from_r(r, pp, 9) == predicted_topk_mask(matmul_nt(lq, lk), 9));
        CHECK(throws<ShapeError>([&] { gpu::predicted_topk_mask(Matrix(Lx, dm + 1), pp, 3); }));
    }

    STEP("routing");
    // per-head sparse_attention routed by mask structure: band-shared
    // (COLVEC) and 32 x 32 block masks reach the tensor-core kernels; same
    // result as the reference within the bf16 bar
    {
        const size_t Lb = 256;
        Matrix qb = bf16_normal(Lb, d, rng), kb = bf16_normal(Lb, d, rng), vb = bf16_normal(Lb, d, rng);
        SparseMask band(Lb), blk(Lb);
        for (size_t i = 0; i < Lb; ++i) {
            for (uint32_t j = (i / 8) % 5; j < Lb; j += 7) band.kept[i].push_back(j);
            // block row ib keeps blocks ib and (ib + 3) % 8
            for (uint32_t b : {static_cast<uint32_t>(i / 32), static_cast<uint32_t>((i / 32 + 3) % 8)})
                for (uint32_t j = b * 32; j < b * 32 + 32; ++j) blk.kept[i].push_back(j);
            std::sort(blk.kept[i].begin(), blk.kept[i].end());
        }
        for (const SparseMask* m : {&band, &blk}) {
            Matrix zg = gpu::sparse_attention(qb, kb, vb, *m, true);
            Matrix zr = spmm(sparse_softmax(sddmm(qb, kb, *m, true)), vb);
            CHECK(max_abs_diff(zg, zr) <= 1e-2 * max_abs(zr));
        }
    }

    STEP("unfused operators");
    // sddmm / sparse_softmax / spmm separately (P/include/dsattn/sparse.hpp:47-55):
    // bit-identical to the reference's scalar kernels (fma per term in index
    // order), within a few ulps of its AVX2 kernels; softmax to the ulp of exp
    {
        SparseMask e = r;  // row top-k mask from above; one empty row, one single-entry row
        e.kept[3].clear();
        e.kept[5] = {7};
        for (kernels::Isa isa : {kernels::Isa::scalar, kernels::Isa::avx2}) {
            kernels::force_isa(isa);
            const bool exact = isa == kernels::Isa::scalar;
            for (bool scale : {true, false}) {
                SparseScores sr = sddmm(q, kk, e, scale), sg = gpu::sddmm(q, kk, e, scale);
                CHECK(sg.row_offsets == sr.row_offsets && sg.mask == sr.mask && sg.values.size() == sr.values.size());
                double ds = 0, ms = 0;
                for (size_t i = 0; i < sr.values.size(); ++i) {
                    ds = std::max(ds, std::abs(sg.values[i] - sr.values[i]));
                    ms = std::max(ms, std::abs(sr.values[i]));
                }
                CHECK(exact ? ds == 0.0 : ds <= 1e-13 * ms);
                // the softmax and the product on the SAME scores, so each operator is checked alone
                SparseWeights wr = sparse_softmax(sr), wg = gpu::sparse_softmax(sr);
                CHECK(wg.empty_row == wr.empty_row && wg.empty_row[3] == 1 && wg.row_offsets == wr.row_offsets);
                double dw = 0;
                for (size_t i = 0; i < wr.values.size(); ++i) dw = std::max(dw, std::abs(wg.values[i] - wr.values[i]));
                CHECK(dw <= 4e-16);
                CHECK(wg.values[wg.row_offsets[5]] == 1.0);
                Matrix zr = spmm(wr, v), zg = gpu::spmm(wr, v);
                CHECK(exact ? max_abs_diff(zg, zr) == 0.0 : max_abs_diff(zg, zr) <= 1e-13 * max_abs(zr));
                bool zero = true;
                for (size_t j = 0; j < d; ++j) zero &= zg(3, j) == 0.0;
                CHECK(zero);
                // the chain on the device end to end == the fused kernel within the f32 bar
                Matrix zc = gpu::spmm(gpu::sparse_softmax(gpu::sddmm(q, kk, e, scale)), v);
                CHECK(max_abs_diff(zc, zr) <= 1e-12 * std::max(1.0, max_abs(zr)));
            }
        }
        kernels::reset_isa();
        OpCounters before = op_counters();  // the device operators do not touch the host counters
        (void)gpu::sddmm(q, kk, e, true);
        CHECK(op_counters().sddmm_mults == before.sddmm_mults);
        CHECK(throws<ShapeError>([&] { gpu::sddmm(q, Matrix(L, d + 1), e, true); }));
        CHECK(throws<ShapeError>([&] { gpu::sddmm(Matrix(L + 1, d), kk, e, true); }));
        CHECK(throws<ShapeError>([&] { gpu::spmm(sparse_softmax(sddmm(q, kk, e, true)), Matrix(L + 1, d)); }));
        SparseMask none(L);  // nothing kept anywhere: empty values, every row flagged, zero output
        SparseWeights wn = gpu::sparse_softmax(gpu::sddmm(q, kk, none, true));
        CHECK(wn.values.empty() && std::count(wn.empty_row.begin(), wn.empty_row.end(), 1) == static_cast<long>(L));
        CHECK(max_abs(gpu::spmm(wn, v)) == 0.0);
    }

    STEP("row_topk_indices / oracle_topk_mask / prediction_accuracy");
    {
        Rng trng(5);
        // non-square, heavy ties (values in {-2..2}), -0 / +0, keep = 1, cols, in between
        Matrix t(37, 91);
        for (size_t i = 0; i < t.size(); ++i) t.raw()[i] = std::floor(trng.normal() * 1.2);
        t.raw()[3] = -0.0;
        t.raw()[4] = 0.0;
        for (size_t keep_n : {size_t{1}, size_t{7}, size_t{90}, size_t{91}})
            CHECK(gpu::row_topk_indices(t, keep_n) == row_topk_indices(t, keep_n));
        CHECK(throws<ParamError>([&] { gpu::row_topk_indices(t, 0); }));
        CHECK(throws<ParamError>([&] { gpu::row_topk_indices(t, 92); }));
        // the oracle mask of the exact scores, and the prediction accuracy of the predicted mask against it
        Matrix sraw = matmul_nt(q, kk);
        SparseMask om = oracle_topk_mask(sraw, 17), og = gpu::oracle_topk_mask(sraw, 17);
        CHECK(og == om);
        CHECK(throws<ShapeError>([&] { gpu::oracle_topk_mask(t, 3); }));
        CHECK(gpu::prediction_accuracy(r, om) == prediction_accuracy(r, om));
        CHECK(gpu::prediction_accuracy(om, om) == 1.0);
        SparseMask shorter = om;
        shorter.kept[2].pop_back();
        CHECK(throws<ParamError>([&] { gpu::prediction_accuracy(shorter, om); }));
        CHECK(throws<ParamError>([&] { gpu::prediction_accuracy(SparseMask(L), SparseMask(L)); }));
        CHECK(throws<ParamError>([&] { gpu::prediction_accuracy(SparseMask(L), SparseMask(L + 1)); }));
    }

    STEP("mask generators on a caller-held dense S~");
    {
        // the reference's own signatures (maskgen.hpp:14-30): colvec_mask (sum |s~| per band, both
        // orientations, ragged last band) and threshold_mask (raw and post-softmax, f64 and f32)
        Rng mrng(19);
        const size_t l = 203;
        Matrix sm(l, l);
        for (size_t i = 0; i < sm.size(); ++i) sm.raw()[i] = std::floor(mrng.normal() * 3.0);  // ties
        for (ColVecSpec spec : {ColVecSpec{8, VecOrientation::col}, ColVecSpec{5, VecOrientation::col},
                                ColVecSpec{1, VecOrientation::col}, ColVecSpec{8, VecOrientation::row},
                                ColVecSpec{300, VecOrientation::col}})
            for (double sp : {0.9, 0.5, 0.01})
                CHECK(gpu::colvec_mask(sm, spec, sp) == colvec_mask(sm, spec, sp));
        CHECK(throws<ParamError>([&] { gpu::colvec_mask(sm, ColVecSpec{0, VecOrientation::col}, 0.5); }));
        CHECK(throws<ParamError>([&] { gpu::colvec_mask(sm, ColVecSpec{8, VecOrientation::col}, 1.0); }));
        CHECK(throws<ShapeError>([&] { gpu::colvec_mask(Matrix(4, 5), ColVecSpec{2, VecOrientation::col}, 0.5); }));
        Matrix sf = random_normal(l, l, 0.0, 2.0, mrng);
        for (double th : {-1.0, 0.0, 2.5, 100.0}) CHECK(gpu::threshold_mask(sf, th, false) == threshold_mask(sf, th, false));
        for (double th : {1e-4, 1.0 / l, 0.05, 0.9}) {
            CHECK(gpu::threshold_mask(sf, th, true) == threshold_mask(sf, th, true));
            Matrix s32 = sf.as_precision(Precision::f32);
            CHECK(gpu::threshold_mask(s32, th, true) == threshold_mask(s32, th, true));
        }
        SparseMask te = gpu::threshold_mask(sf, 0.9, true);
        CHECK(te.has_empty_rows() == threshold_mask(sf, 0.9, true).has_empty_rows());
        CHECK(throws<ParamError>([&] { gpu::threshold_mask(sf, std::nan(""), false); }));
        CHECK(throws<ShapeError>([&] { gpu::threshold_mask(Matrix(4, 5), 0.1, false); }));
    }

    STEP("predictor precision rule");
    // combine() (P/include/dsattn/matrix.hpp:90-93): a product is f32 only when
    // both operands are.  The ToyModel case -- f32 activations and W~, f64
    // ternary P -- runs the whole chain in f64; all-f32 rounds every product.
    {
        Rng prng(77);
        auto proj = std::make_shared<ProjectionMatrix>(init_projection(d, 16, 9));  // f64
        Matrix xf = bf16_normal(96, d, prng).as_precision(Precision::f32);
        PredictorParams pp = random_predictor_params(proj, 0.3, prng, QuantSpec{4}, Precision::f32);
        auto ref_mask = [&](const PredictorParams& a, const Matrix& x) {
            Matrix rr = matmul(x, a.proj->p);
            Matrix xq = matmul(rr, a.wq), xk = matmul(rr, a.wk);
            auto lv = [&](const Matrix& m) {
                Matrix qt = quantize(m, a.quant);
                const double sc = max_abs(m) / 7.0;
                Matrix o(qt.rows(), qt.cols());
                for (size_t i = 0; i < qt.size(); ++i) o.raw()[i] = sc == 0 ? 0 : std::lround(qt.data()[i] / sc);
                return o;
            };
            return predicted_topk_mask(matmul_nt(lv(xq), lv(xk)), 11);
        };
        CHECK(gpu::predicted_topk_mask(xf, pp, 11) == ref_mask(pp, xf));            // f32 x, f64 P, f32 W~
        auto proj32 = std::make_shared<ProjectionMatrix>(*proj);
        proj32->p = proj->p.as_precision(Precision::f32);
        PredictorParams pp32 = pp;
        pp32.proj = proj32;
        CHECK(gpu::predicted_topk_mask(xf, pp32, 11) == ref_mask(pp32, xf));        // everything f32
        PredictorParams mixed = pp32;
        mixed.wq = pp.wq.as_precision(Precision::f64);
        mixed.wk = pp.wk.as_precision(Precision::f64);
        CHECK(throws<ParamError>([&] { gpu::predicted_topk_mask(xf, mixed, 11); }));  // stage one rounds, stage two not
    }

    // reference exception types (P/include/dsattn/errors.hpp)
    CHECK(throws<ParamError>([&] { gpu::predicted_topk_mask(q, kk, p, QuantSpec{4}, 0); }));
    CHECK(throws<ParamError>([&] { gpu::predict(q, kk, p, QuantSpec{3}); }));
    CHECK(throws<ShapeError>([&] { gpu::sparse_attention(q, kk, Matrix(L + 1, d), r, true); }));

    std::printf("shim: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
