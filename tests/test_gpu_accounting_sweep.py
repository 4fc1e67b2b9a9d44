"""Accounting on the seeded random configurations of test_gpu_sweep: for each
GPU-produced mask, dsa_counters == the reference OpCounters of sddmm ->
sparse_softmax -> spmm on the same mask, and dsa_dataflow_trace == the
reference dataflow::simulate (three schedules, two band heights) -- every
mask layout, ragged L, empty rows, keep from 1 to L."""
import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import load_preset, ops
from test_gpu_shapes import BASE
from test_gpu_sweep import _cases

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("idx,case", list(enumerate(_cases(24, 777))), ids=lambda v: str(v) if isinstance(v, int) else v[0])
def test_counters_and_dataflow_match_reference(idx, case, reference):
    mode, L, d, k, bits, dtype, scope, extra = case
    if L > 1500:
        L = 1500 - (idx % 7)  # the reference simulate is O(nnz log) per band on the host: keep it short
        for key in ("keep", "cap"):
            if key in extra:
                extra = dict(extra, **{key: min(extra[key], L)})
        if mode == "block":
            extra = dict(extra, keep=min(extra["keep"], -(-L // extra["block"])))
    npairs = 2
    p = load_preset(BASE[mode]).replace(L=L, d=d, k=k, bits=bits, dtype=dtype, quant_scope=scope,
                                        round_proj_f32=(dtype == "f32"), seed=5 + L, batch=npairs, heads=1, **extra)
    q, k_, v, P = ops.generate(p, npairs=npairs)
    dev = torch.device("cuda:0")
    qd, kd, Pd = (t.to(dev) for t in (q, k_, P))
    mask = ops.select(p, ops.predict(p, qd, kd, Pd))
    torch.cuda.synchronize()
    rows = ops.mask_rows(p, mask, npairs)
    cnt = ops.counters(p, mask, npairs)
    tot = np.zeros(3, np.uint64)
    empty = 0
    csr = []
    for pr in range(npairs):
        rp, cols = ops.to_csr(rows[pr])
        csr.append((rp, cols))
        _, er, c = reference.sparse_attention(q[pr].double().numpy(), k_[pr].double().numpy(),
                                              v[pr].double().numpy(), rp, cols, True, p.dtype == "f32")
        tot += c
        empty += int(er.sum())
    assert [cnt["sddmm_mults"], cnt["spmm_mults"], cnt["softmax_exps"]] == tot.tolist()
    assert cnt["nnz"] == int(tot[2])
    if p.mask_mode == "threshold":
        assert cnt["empty_rows"] == empty
    for sched in ("row_by_row", "row_parallel", "row_parallel_reordered"):
        for band in (3, 8):
            f, i = ops.dataflow_trace(p, mask, npairs, sched, band)
            for pr in range(npairs):
                rf, ri = reference.dataflow_simulate(csr[pr][0], csr[pr][1], sched, band)
                assert (int(f[pr]), int(i[pr])) == (rf, ri), f"{sched} band {band} pair {pr}"
