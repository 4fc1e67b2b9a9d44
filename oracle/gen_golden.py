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
                      or the max-pooled colvec composition
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
    if p.mask_mode == "row_topk":
        m = ref.topk_mask(S, p.keep)
        rows = [m[i] for i in range(p.L)]
    else:
        m = ref.colvec_maxpool_mask(S, p.vec_v, p.keep)
        rows = [m[i // p.vec_v] for i in range(p.L)]
    rp = np.zeros(p.L + 1, np.uint64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    cols = np.concatenate(rows).astype(np.uint32)
    z, er, cnt = ref.sparse_attention(qn, kn, vn, rp, cols, True, f32)
    raw = {"q": q[0].view(torch.int16).numpy() if p.dtype == "bf16" else q[0].numpy(),
           "k": k[0].view(torch.int16).numpy() if p.dtype == "bf16" else k[0].numpy(),
           "v": v[0].view(torch.int16).numpy() if p.dtype == "bf16" else v[0].numpy()}
    np.savez_compressed(OUT / f"{name}.npz", **raw, P=P.numpy(), lq=lq.astype(np.int8),
                        lk=lk.astype(np.int8), sq=np.float64(sq), sk=np.float64(sk),
                        mask=m.astype(np.uint16), z=z, counters=cnt,
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


if __name__ == "__main__":
    main()
