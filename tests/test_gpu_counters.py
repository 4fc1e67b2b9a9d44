"""Accounting on GPU-produced masks against the reference:

* dsa_counters == the reference OpCounters (P/src/sparse.cpp:13-16, 51, 75,
  89) accumulated by sddmm -> sparse_softmax -> spmm over the SAME mask
  (every mode: row lists, band lists, block lists, ragged CSR with empty
  rows);
* dsa_prediction_accuracy (device) == the reference prediction_accuracy
  (P/src/maskgen.cpp:94-107) of the GPU predicted mask against the
  reference oracle_topk_mask on the true scores Q K^T (P/src/maskgen.cpp:
  11-16), and it raises ParamError on unequal per-row counts."""
import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import load_preset, ops
from paper_2110_11299_b200.errors import ParamError
from test_gpu_parity import run_gpu

pytestmark = pytest.mark.gpu

CASES = [("c1_bert_base", {"L": 512, "keep": 26}), ("c2_vector", {"L": 1024, "keep": 51}),
         ("c3_block", {"L": 1024, "keep": 5}), ("c4_threshold", {"L": 1200, "cap": 40}),
         ("c4_threshold", {"L": 700, "cap": 50, "frac_num": 1, "frac_den": 400})]


@pytest.mark.parametrize("name,over", CASES)
def test_counters_match_reference_opcounters(name, over, reference):
    p = load_preset(name).replace(**over)
    npairs = 2
    sub, (q, k, v, P), lv, mask, z = run_gpu(p, npairs)
    cnt = ops.counters(sub, mask, npairs)
    rows = ops.mask_rows(sub, mask, npairs)
    tot = np.zeros(3, np.uint64)
    empty = 0
    for pr in range(npairs):
        rp, cols = ops.to_csr(rows[pr])
        _, er, c = reference.sparse_attention(q[pr].double().numpy(), k[pr].double().numpy(),
                                              v[pr].double().numpy(), rp, cols, True, sub.dtype == "f32")
        tot += c
        empty += int(er.sum())
    assert [cnt["sddmm_mults"], cnt["spmm_mults"], cnt["softmax_exps"]] == tot.tolist()
    assert cnt["nnz"] == int(tot[2])
    if sub.mask_mode == "threshold":
        assert cnt["empty_rows"] == empty


def test_prediction_accuracy_matches_reference(reference):
    p = load_preset("c1_bert_base").replace(L=512, keep=26, quant_scope="tensor")
    npairs = 2
    sub, (q, k, v, P), lv, mask, z = run_gpu(p, npairs)
    dev = torch.device("cuda:0")
    orc = []
    for pr in range(npairs):
        qn, kn = q[pr].double().numpy(), k[pr].double().numpy()
        s = reference.project(qn, np.ascontiguousarray(kn.T))  # matmul(q, k^T) = matmul_nt(q, k)
        orc.append(reference.topk_mask(s, p.keep))            # oracle_topk_mask(s_raw, keep)
    omask = ops.Mask("row_topk", torch.from_numpy(np.concatenate([o.ravel() for o in orc]).astype(np.int32)).to(dev),
                     None, None)
    acc = ops.prediction_accuracy(sub, mask, omask, npairs)
    rows = ops.mask_rows(sub, mask, npairs)
    rp_p, c_p = ops.to_csr([r for pr in rows for r in pr])
    rp_o, c_o = ops.to_csr([o[i] for o in orc for i in range(p.L)])
    want = reference.prediction_accuracy(rp_p, c_p, rp_o, c_o)
    assert acc == want and 0.0 < acc < 1.0
    # the same masks as global CSR give the same value; unequal per-row
    # counts -> ParamError, as the reference
    thr = sub.replace(mask_mode="threshold", cap=p.L)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).astype(dt)).to(dev)  # noqa: E731
    pm = ops.Mask("threshold", t(c_p, np.int32), t(rp_p, np.int64), None)
    om = ops.Mask("threshold", t(c_o, np.int32), t(rp_o, np.int64), None)
    assert ops.prediction_accuracy(thr, pm, om, npairs) == want
    rp_bad = rp_o.astype(np.int64).copy()
    rp_bad[1:] -= 1
    c_bad = np.delete(c_o, int(rp_o[1]) - 1)
    with pytest.raises(ParamError):
        ops.prediction_accuracy(thr, pm, ops.Mask("threshold", t(c_bad, np.int32), t(rp_bad, np.int64), None), npairs)
