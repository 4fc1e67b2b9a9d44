"""Edge inputs of the projection + quantisation (P/src/predictor.cpp:34-45,
P/src/kernels/scalar.cpp:11-17,60-68) on the tensor-core path:

* every projected value exactly on a .5 rounding boundary -- no level can be
  certified from the fp32 tensor-core value, so the deferred-recompute list
  overflows (capacity = a quarter of the levels) and the in-place fallback
  recomputes the rest with the reference's fp64 chain: levels and scale
  must still equal the reference's round-half-away;
* an all-zero tensor: scale 0 and every level 0 (the amax == 0 guard,
  P/src/predictor.cpp:39)."""
import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import load_preset, ops

pytestmark = pytest.mark.gpu


def _levels(p, q, k, P):
    dev = torch.device("cuda:0")
    lv = ops.predict(p, q.to(dev), k.to(dev), P.to(dev))
    torch.cuda.synchronize()
    return (ops.levels_rows(lv.lq).float().cpu().numpy().astype(np.int32),
            ops.levels_rows(lv.lk).float().cpu().numpy().astype(np.int32), lv.sq.cpu().numpy(), lv.sk.cpu().numpy())


@pytest.mark.parametrize("bits", [4, 2])
def test_all_levels_on_rounding_boundaries(bits, oracle):
    p = load_preset("c2_vector").replace(batch=2, heads=1, L=512, keep=26, bits=bits)
    qmax = (1 << (bits - 1)) - 1
    rng = np.random.default_rng(3)
    # P = [I_k; 0]: Q.P is exactly the first k columns of Q
    P = np.zeros((p.d, p.k), np.float32)
    P[np.arange(p.k), np.arange(p.k)] = 1.0
    x = rng.integers(-qmax, qmax, size=(2, p.L, p.d)).astype(np.float64) + 0.5  # n + 0.5 with |.| <= qmax - 0.5
    x[:, 0, 0] = qmax  # amax = qmax -> s = 1: every other value sits exactly on a .5 boundary
    q = torch.from_numpy(x).to(torch.bfloat16)
    k = torch.from_numpy(-x).to(torch.bfloat16)
    lq, lk, sq, sk = _levels(p, q, k, torch.from_numpy(P))
    for pr in range(2):
        rq, s_q = oracle.levels(q[pr].double().numpy(), P.astype(np.float64), bits)
        rk, s_k = oracle.levels(k[pr].double().numpy(), P.astype(np.float64), bits)
        assert s_q == 1.0 and s_k == 1.0
        assert np.array_equal(lq[pr], rq) and np.array_equal(lk[pr], rk)
        assert sq[pr] == s_q and sk[pr] == s_k


def test_zero_tensor_gives_zero_scale_and_levels():
    p = load_preset("c2_vector").replace(batch=1, heads=1, L=256, keep=13)
    q = torch.zeros((1, p.L, p.d), dtype=torch.bfloat16)
    k = torch.randn((1, p.L, p.d)).to(torch.bfloat16)
    _, P = ops.generate(p, npairs=1)[2:]
    lq, lk, sq, sk = _levels(p, q, k, P)
    assert sq[0] == 0.0 and not lq.any()
    assert sk[0] > 0.0 and lk.any()
