"""The reference's dataflow fetch-count model (dataflow::simulate,
P/src/dataflow.cpp:10-62; the cost model SURVEY 8(f) item 4 names) on
device masks of every layout, against the reference itself on the same
masks: operand_fetches and pe_idle_steps per (b,h) pair, for the three
schedules and several band heights (incl. ragged last bands)."""
import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import load_preset, ops

pytestmark = pytest.mark.gpu

CASES = [
    ("c1_bert_base", {"L": 512, "keep": 26}),
    ("c2_vector", {"L": 1000, "keep": 50}),
    ("c3_block", {"L": 1000, "keep": 5}),
    ("c4_threshold", {"L": 1500, "cap": 60}),
    ("c0_smoke", {}),
]


@pytest.mark.parametrize("name,over", CASES, ids=[c[0] for c in CASES])
def test_dataflow_matches_reference(name, over, reference):
    npairs = 1 if name == "c0_smoke" else 2
    p = load_preset(name).replace(batch=npairs, heads=1, **over)
    q, k, v, P = ops.generate(p, npairs=npairs)
    dev = torch.device("cuda:0")
    qd, kd, Pd = (t.to(dev) for t in (q, k, P))
    mask = ops.select(p, ops.predict(p, qd, kd, Pd))
    torch.cuda.synchronize()
    rows = ops.mask_rows(p, mask, npairs)
    for sched in ("row_by_row", "row_parallel", "row_parallel_reordered"):
        for band in (1, 4, 7, 8, 32):
            f, i = ops.dataflow_trace(p, mask, npairs, sched, band)
            for pr in range(npairs):
                rp, cols = ops.to_csr(rows[pr])
                rf, ri = reference.dataflow_simulate(rp, cols, sched, band)
                assert (int(f[pr]), int(i[pr])) == (rf, ri), f"{name} {sched} band {band} pair {pr}"


def test_dataflow_rejects_bad_band():
    from paper_2110_11299_b200 import errors
    p = load_preset("c2_vector").replace(batch=1, heads=1, L=256, keep=13)
    q, k, v, P = ops.generate(p, npairs=1)
    dev = torch.device("cuda:0")
    mask = ops.select(p, ops.predict(p, q.to(dev), k.to(dev), P.to(dev)))
    with pytest.raises(errors.ParamError):
        ops.dataflow_trace(p, mask, 1, "row_parallel", 0)
