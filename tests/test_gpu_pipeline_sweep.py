"""dsa_pipeline (the one-call entry point bench.py times) against the three
phase calls on the seeded random configurations of test_gpu_sweep: the same
kernels run in both, so Z and the mask must be IDENTICAL bit for bit, with
and without a caller mask, on a side stream, and with 3 and 5 pairs (odd pair
counts exercise the workspace offsets of every per-pair scratch region)."""
import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import load_preset, ops
from test_gpu_shapes import BASE
from test_gpu_sweep import _cases

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("idx,case", list(enumerate(_cases(36, 4242))), ids=lambda v: str(v) if isinstance(v, int) else v[0])
def test_pipeline_equals_phases(idx, case):
    mode, L, d, k, bits, dtype, scope, extra = case
    npairs = 3 if idx % 2 else 5
    p = load_preset(BASE[mode]).replace(L=L, d=d, k=k, bits=bits, dtype=dtype, quant_scope=scope,
                                        round_proj_f32=(dtype == "f32"), seed=99 + L, batch=npairs, heads=1, **extra)
    q, k_, v, P = ops.generate(p, pair0=idx, npairs=npairs)
    dev = torch.device("cuda:0")
    qd, kd, vd, Pd = (t.to(dev) for t in (q, k_, v, P))
    lv = ops.predict(p, qd, kd, Pd)
    mask = ops.select(p, lv)
    z = ops.sparse_attention(p, qd, kd, vd, mask)
    torch.cuda.synchronize()

    s = torch.cuda.Stream()
    with_mask = ops.Pipeline(p, pairs=npairs, device=dev, keep_mask=True)
    s.wait_stream(torch.cuda.current_stream())
    z1 = with_mask(qd, kd, vd, Pd, stream=s)
    s.synchronize()
    assert torch.equal(z1, z), "pipeline (caller mask) Z differs from the phase calls"
    r0, r1 = ops.mask_rows(p, mask, npairs), ops.mask_rows(p, with_mask.mask, npairs)
    for pr in range(npairs):
        for i in range(L):
            assert np.array_equal(r0[pr][i], r1[pr][i]), (pr, i)
    if mask.empty_rows is not None and with_mask.mask.empty_rows is not None:
        assert torch.equal(mask.empty_rows[: npairs * L], with_mask.mask.empty_rows[: npairs * L])

    no_mask = ops.Pipeline(p, pairs=npairs, device=dev)
    z2 = no_mask(qd, kd, vd, Pd)
    torch.cuda.synchronize()
    assert torch.equal(z2, z), "pipeline (internal mask) Z differs from the phase calls"
