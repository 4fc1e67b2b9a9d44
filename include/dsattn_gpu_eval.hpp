// the reference's product caller routed through the GPU
// path.  The reference's `evaluate` (P/src/trainer.cpp:422-469) calls
// `forward_batch` (P/src/trainer.cpp:120-294), whose DSA branch predicts
// S~ = quant(R W~_Q) quant(R W~_K)^T per head (:173-175), selects
// `predicted_topk_mask(S~, keep)` (:190-195) and then runs a DENSE softmax
// with an additive mask (:218-221) followed by A V (:235).  Here the same
// inference forward keeps every non-attention operator on the reference's
// own Tape (embedding, layer norm, the per-head weight matmuls, W_O, the
// feed-forward sublayer, the classifier read-out) and replaces
//   * the mask: `dsattn::gpu::predicted_topk_mask(h, PredictorParams, keep)`
//     -- dsa_predict_wtilde + dsa_select, bit-identical levels and masks;
//   * the attention: `dsattn::gpu::sparse_attention` -- SDDMM -> sparse
//     softmax -> SpMM over the kept positions only (the paper's deployment
//     target), per head in the tensors' own precision, or for the whole
//     layer in one bf16 tensor-core call (dsa_project_qkv + one batched
//     attention).
// Header-only host code above the C ABI; needs the reference's trainer /
// model / autodiff / task headers and objects at link time (it is the patch
// a maintainer would apply inside trainer.cpp, kept outside the reference).
// Inference only: no gradients (the trainer's autodiff stays out of scope).
#pragma once

#include <cmath>
#include <string>
#include <vector>

#include "dsattn/autodiff.hpp"
#include "dsattn/linalg.hpp"
#include "dsattn/model.hpp"
#include "dsattn/task.hpp"
#include "dsattn/trainer.hpp"
#include "dsattn_gpu.hpp"

namespace dsattn::gpu {

enum class EvalAttention {
    sparse_per_head,  // Q/K/V by the reference matmul, gpu::sparse_attention per head (f32 / bf16 by the tensors)
    sparse_layer,     // the layer-level gpu::sparse_attention(x, params, masks): bf16 tensor cores
    reference_dense,  // GPU masks only; the reference's own additive-mask dense softmax (bit-identical forward)
};

struct GpuEvalOptions {
    double sparsity = 0.9;
    int bits_override = -1;  // as EvalOptions::bits_override; the device predictor needs 2, 4 or 8 bits
    EvalAttention attention = EvalAttention::sparse_per_head;
    bool capture_masks = false;  // keep every sample's masks and predictor inputs in the result
    // evaluate(collect_stats = true) (P/src/trainer.cpp:204-207, 459-463): the predicted mask's
    // accuracy against oracle_topk_mask(Q K^T, keep), mean over heads and samples per layer --
    // the oracle mask (dsa_row_topk_f64) and the comparison (dsa_prediction_accuracy) on the device
    bool collect_stats = false;
};

struct GpuEvalResult {
    double accuracy = 0.0;
    std::vector<uint32_t> predictions;                          // argmax per sample
    std::vector<std::vector<double>> logits;                    // per sample
    std::vector<std::vector<std::vector<SparseMask>>> masks;    // [sample][layer][head] when captured
    std::vector<std::vector<Matrix>> layer_inputs;              // [sample][layer]: the predictor input h, when captured
    std::vector<double> pred_acc_per_layer;                     // with collect_stats
};

namespace detail {

inline SparseMask full_mask(size_t l) {
    SparseMask m;
    m.l = l;
    m.kept.resize(l);
    for (auto& row : m.kept) {
        row.resize(l);
        for (size_t j = 0; j < l; ++j) row[j] = static_cast<uint32_t>(j);
    }
    return m;
}

}  // namespace detail

// One sample through the model (P/src/trainer.cpp:154-262 with dsa = true,
// MaskKind::predicted, no gradients); returns the logits row.
inline std::vector<double> forward_sample(ToyModel& model, const TaskSpec& spec, const Sample& sample,
                                          const GpuEvalOptions& opts,
                                          std::vector<std::vector<SparseMask>>* masks_out = nullptr,
                                          std::vector<Matrix>* layer_inputs_out = nullptr,
                                          std::vector<double>* pred_acc_sum = nullptr) {
    const ModelConfig& cfg = model.config();
    const size_t l = cfg.seq_len;
    if (spec.l != l || spec.vocab != cfg.vocab) throw ShapeError("forward_batch: task/model shape mismatch");
    if (sample.tokens.size() != l) throw ShapeError("forward_batch: sample length != l");
    const size_t keep = keep_per_row(l, opts.sparsity);
    const QuantSpec quant{opts.bits_override >= 0 ? opts.bits_override : cfg.pred_bits};
    quant.validate();
    if (quant.bits != 2 && quant.bits != 4 && quant.bits != 8)
        throw ParamError("dsattn::gpu::evaluate: the device predictor needs 2-, 4- or 8-bit levels");
    const double inv_sqrt_dk = 1.0 / std::sqrt(static_cast<double>(cfg.d_head()));

    ad::Tape tape(false);
    auto par = [&](const std::string& name) { return tape.constant(model.param(name).value); };
    ad::Var x = tape.add(tape.embedding(par("emb"), sample.tokens), par("pos"));
    if (masks_out) masks_out->assign(cfg.layers, std::vector<SparseMask>(cfg.heads));
    for (size_t layer = 0; layer < cfg.layers; ++layer) {
        const std::string lp = "layer" + std::to_string(layer) + ".";
        ad::Var h = tape.layer_norm(x, par(lp + "ln1.g"), par(lp + "ln1.b"));
        const Matrix hv = tape.value(h);  // a copy: later tape ops may reallocate the node table
        if (layer_inputs_out) layer_inputs_out->push_back(hv);
        // masks: the device predictor on the layer input (R = h P once per call)
        std::vector<SparseMask> masks(cfg.heads);
        for (size_t hd = 0; hd < cfg.heads; ++hd) {
            const std::string hp = lp + "h" + std::to_string(hd) + ".";
            if (keep >= l) {  // sparsity 0: the reference takes the dense path
                masks[hd] = detail::full_mask(l);
                continue;
            }
            PredictorParams pp;
            pp.proj = model.projections()[layer];
            pp.wq = model.param(hp + "pred.wq").value;
            pp.wk = model.param(hp + "pred.wk").value;
            pp.quant = quant;
            masks[hd] = gpu::predicted_topk_mask(hv, pp, keep);
        }
        if (masks_out) (*masks_out)[layer] = masks;
        if (pred_acc_sum && keep < l) {
            for (size_t hd = 0; hd < cfg.heads; ++hd) {
                const std::string hp = lp + "h" + std::to_string(hd) + ".";
                const Matrix s_raw = matmul_nt(matmul(hv, model.param(hp + "wq").value),
                                               matmul(hv, model.param(hp + "wk").value));  // unscaled, :170
                (*pred_acc_sum)[layer] += gpu::prediction_accuracy(masks[hd], gpu::oracle_topk_mask(s_raw, keep));
            }
        }

        ad::Var z;
        if (opts.attention == EvalAttention::sparse_layer) {
            AttentionParams ap;
            ap.scale = cfg.scale_scores;
            for (size_t hd = 0; hd < cfg.heads; ++hd) {
                const std::string hp = lp + "h" + std::to_string(hd) + ".";
                ap.wq.push_back(model.param(hp + "wq").value);
                ap.wk.push_back(model.param(hp + "wk").value);
                ap.wv.push_back(model.param(hp + "wv").value);
            }
            ap.heads = cfg.heads;
            z = tape.constant(gpu::sparse_attention(hv, ap, std::span<const SparseMask>(masks)));
        } else {
            std::vector<ad::Var> head_outputs;
            for (size_t hd = 0; hd < cfg.heads; ++hd) {
                const std::string hp = lp + "h" + std::to_string(hd) + ".";
                ad::Var q = tape.matmul(h, par(hp + "wq"));
                ad::Var k = tape.matmul(h, par(hp + "wk"));
                ad::Var v = tape.matmul(h, par(hp + "wv"));
                if (opts.attention == EvalAttention::reference_dense) {
                    ad::Var s_raw = tape.matmul_nt(q, k);
                    ad::Var s = cfg.scale_scores ? tape.scale(s_raw, inv_sqrt_dk) : s_raw;
                    ad::Var a = keep >= l ? tape.softmax_rows(s)
                                          : tape.softmax_rows_masked(s, masks[hd], cfg.mask_constant);
                    head_outputs.push_back(tape.matmul(a, v));
                } else {
                    head_outputs.push_back(tape.constant(
                        gpu::sparse_attention(tape.value(q), tape.value(k), tape.value(v), masks[hd], cfg.scale_scores)));
                }
            }
            z = cfg.heads == 1 ? head_outputs[0] : tape.concat_cols(head_outputs);
        }
        x = tape.add(x, tape.matmul(z, par(lp + "wo")));
        ad::Var h2 = tape.layer_norm(x, par(lp + "ln2.g"), par(lp + "ln2.b"));
        ad::Var f = tape.tanh_act(tape.add_row_broadcast(tape.matmul(h2, par(lp + "ffn.w1")), par(lp + "ffn.b1")));
        x = tape.add(x, tape.add_row_broadcast(tape.matmul(f, par(lp + "ffn.w2")), par(lp + "ffn.b2")));
    }
    ad::Var xf = tape.layer_norm(x, par("lnf.g"), par("lnf.b"));
    ad::Var readout = tape.row(xf, sample.marker_pos);
    ad::Var logits = tape.add_row_broadcast(tape.matmul(readout, par("head.w")), par("head.b"));
    const Matrix& lg = tape.value(logits);
    std::vector<double> out(lg.cols());
    for (size_t j = 0; j < lg.cols(); ++j) out[j] = lg(0, j);
    return out;
}

// evaluate(model, task, {dsa = true, MaskKind::predicted, sparsity, bits})
// (P/src/trainer.cpp:422-469) through the GPU path: accuracy = the fraction
// of samples whose argmax logit (first maximum, :252-255) is the label.
inline GpuEvalResult evaluate(ToyModel& model, const ToyTask& task, const GpuEvalOptions& opts) {
    GpuEvalResult res;
    size_t correct = 0;
    for (const Sample& s : task.samples) {
        std::vector<std::vector<SparseMask>> masks;
        std::vector<Matrix> inputs;
        if (opts.collect_stats && res.pred_acc_per_layer.empty())
            res.pred_acc_per_layer.assign(model.config().layers, 0.0);
        std::vector<double> lg = forward_sample(model, task.spec, s, opts, opts.capture_masks ? &masks : nullptr,
                                                opts.capture_masks ? &inputs : nullptr,
                                                opts.collect_stats ? &res.pred_acc_per_layer : nullptr);
        uint32_t best = 0;
        for (size_t j = 1; j < lg.size(); ++j)
            if (lg[j] > lg[best]) best = static_cast<uint32_t>(j);
        res.predictions.push_back(best);
        res.logits.push_back(std::move(lg));
        if (opts.capture_masks) {
            res.masks.push_back(std::move(masks));
            res.layer_inputs.push_back(std::move(inputs));
        }
        correct += best == s.label;
    }
    for (double& a : res.pred_acc_per_layer)
        a /= static_cast<double>(task.samples.size() * model.config().heads);
    res.accuracy = task.samples.empty() ? 0.0 : static_cast<double>(correct) / static_cast<double>(task.samples.size());
    return res;
}

}  // namespace dsattn::gpu
