"""Generates tests/golden/*.npz from the REFERENCE implementation itself
(oracle/_ref/libdsattn_ref.so, compiled from /root/reference/proj/src).

TEST INFRASTRUCTURE ONLY.  Run in the build container (the reference tree
is not on the GPU box); the fixtures are committed.

    python oracle/gen_golden.py

Each fixture holds the seeded inputs and the reference's outputs:
  * levels / scales : reference matmul + quantize (P/src/linalg.cpp:11-17,
                      P/src/predictor.cpp:34-45), integer levels recovered as
                      lround(q~ / s)
  * mask            : predicted_topk_mask on the exact integer S~ (row top-k),
                      the max-pooled colvec composition, the
                      block-mean composition (O5: ref_block_mask) or the
                      causal softmax threshold + cap (O6:
                      ref_causal_threshold_mask = row_softmax, ">= theta",
                      row_topk_indices)
  * z               : sddmm -> sparse_softmax -> spmm (P/src/sparse.cpp:38-91)
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle.oracle import Reference  # noqa: E402
from paper_2110_11299_b200 import load_preset, ops  # noqa: E402

OUT = ROOT / "tests" / "golden"


def levels(ref, x, P, bits, f32):
    xp = ref.project(x, P, f32)
    lv, s = ref.quantize_levels(xp, bits, f32)
    return lv, s


def case(name, p, ref):
    q, k, v, P = ops.generate(p.replace(batch=1, heads=1), npairs=1)
    f32 = p.dtype == "f32"
    qn, kn, vn, Pn = q[0].double().numpy(), k[0].double().numpy(), v[0].double().numpy(), P.double().numpy()
    lq, sq = levels(ref, qn, Pn, p.bits, f32)
    lk, sk = levels(ref, kn, Pn, p.bits, f32)
    S = (lq.astype(np.int64) @ lk.T.astype(np.int64)).astype(np.float64)
    extra = {}
    if p.mask_mode == "row_topk":
        m = ref.topk_mask(S, p.keep)
        rows = [m[i] for i in range(p.L)]
    elif p.mask_mode == "colvec":
        m = ref.colvec_maxpool_mask(S, p.vec_v, p.keep)
        rows = [m[i // p.vec_v] for i in range(p.L)]
    elif p.mask_mode == "block":
        m = ref.block_mask(lq, lk, p.block, p.keep, p.force_diag)
        rows = [np.concatenate([np.arange(b * p.block, min((b + 1) * p.block, p.L)) for b in m[i // p.block]])
                for i in range(p.L)]
        extra = {"block": np.array([p.block, int(p.force_diag)], np.int64)}
    else:
        c = sq * sk / np.sqrt(float(p.d))
        theta = p.frac_den / (p.frac_num * p.L)
        rp_, cols_ = ref.causal_threshold_mask(lq, lk, c, theta, p.cap, p.causal)
        rows = [cols_[rp_[i]:rp_[i + 1]] for i in range(p.L)]
        m = np.concatenate([rp_.astype(np.int64), cols_.astype(np.int64)])  # rowptr ++ cols
        extra = {"threshold": np.array([p.frac_num, p.frac_den, p.cap, int(p.causal)], np.int64)}
    rp = np.zeros(p.L + 1, np.uint64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    cols = np.concatenate(rows).astype(np.uint32)
    z, er, cnt = ref.sparse_attention(qn, kn, vn, rp, cols, True, f32)
    raw = {"q": q[0].view(torch.int16).numpy() if p.dtype == "bf16" else q[0].numpy(),
           "k": k[0].view(torch.int16).numpy() if p.dtype == "bf16" else k[0].numpy(),
           "v": v[0].view(torch.int16).numpy() if p.dtype == "bf16" else v[0].numpy()}
    np.savez_compressed(OUT / f"{name}.npz", **raw, P=P.numpy(), lq=lq.astype(np.int8),
                        lk=lk.astype(np.int8), sq=np.float64(sq), sk=np.float64(sk),
                        mask=m.astype(np.uint16) if p.mask_mode != "threshold" else m, z=z,
                        counters=cnt, empty_rows=er, **extra,
                        meta=np.array([p.L, p.d, p.k, p.bits, p.keep, p.vec_v, int(f32)], np.int64),
                        mode=np.array(p.mask_mode))
    print(f"{name}: L={p.L} keep={p.keep} ties-resolved mask rows={len(rows)} nnz={int(rp[-1])}")


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    ref = Reference()
    c0 = load_preset("c0_smoke")
    case("c0_smoke_pair0", c0, ref)
    c1 = load_preset("c1_bert_base").replace(L=256, keep=13, quant_scope="tensor", seed=7)
    case("rowtopk_bf16_L256", c1, ref)
    c2 = load_preset("c2_vector").replace(L=512, keep=26, seed=11)
    case("colvec_bf16_L512", c2, ref)
    c3 = load_preset("c3_block").replace(L=256, mask_mode="row_topk", keep=16, seed=13)
    case("rowtopk_int8_d128_L256", c3, ref)
    c3b = load_preset("c3_block").replace(L=512, keep=4, seed=17)
    case("block_int8_d128_L512", c3b, ref)
    c3r = load_preset("c3_block").replace(L=300, d=64, k=16, bits=4, keep=3, seed=19)  # ragged last block
    case("block_bf16_L300_ragged", c3r, ref)
    c4 = load_preset("c4_threshold").replace(L=640, cap=9, seed=23)  # causal, cap binding
    case("threshold_causal_bf16_L640", c4, ref)
    c4n = load_preset("c4_threshold").replace(L=384, causal=False, frac_num=1, frac_den=40, cap=384, seed=29)
    case("threshold_full_bf16_L384", c4n, ref)


if __name__ == "__main__":
    main()
