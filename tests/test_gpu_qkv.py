"""GPU parity of the fused Q/K/V (+ predictor input) projection GEMM
(dsa_project_qkv) against the reference project_qkv
(P/src/attention.cpp:36-46: per-head matmul(X, W), computed here by the
reference's own linalg::matmul in f64 via oracle/_ref and, for the larger
shapes, a plain torch fp32 matmul of the same bf16 operands).

Tolerance (bf16 outputs from fp32 accumulation): max |Y - Y_ref| <= 1e-2 *
max |Y_ref| per head (the BASELINE bf16 bar); R (f32) within 1e-5."""
import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import ops
from paper_2110_11299_b200.errors import ParamError, ShapeError

pytestmark = pytest.mark.gpu


def _inputs(batch, L, dm, heads, dk, dv, npred, seed):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(batch, L, dm, generator=g).to(torch.bfloat16)
    s = 1.0 / dm ** 0.5  # random_attention_params: U(-1/sqrt(d), 1/sqrt(d))
    wq = [((torch.rand(dm, dk, generator=g) * 2 - 1) * s).to(torch.bfloat16) for _ in range(heads)]
    wk = [((torch.rand(dm, dk, generator=g) * 2 - 1) * s).to(torch.bfloat16) for _ in range(heads)]
    wv = [((torch.rand(dm, dv, generator=g) * 2 - 1) * s).to(torch.bfloat16) for _ in range(heads)]
    pm = (torch.randn(dm, npred, generator=g) / max(npred, 1) ** 0.5) if npred else None
    return x, wq, wk, wv, pm


def _run(batch, L, dm, heads, dk, dv, npred, seed=7):
    x, wq, wk, wv, pm = _inputs(batch, L, dm, heads, dk, dv, npred, seed)
    w = ops.pack_qkv_weights(wq, wk, wv, pm)
    q, k, v, r = ops.project_qkv(x.cuda(), w.cuda(), heads, dk, dv, npred)
    torch.cuda.synchronize()
    return x, wq, wk, wv, pm, w, q.cpu(), k.cpu(), v.cpu(), None if r is None else r.cpu()


def _rel(a, b):
    return float((a.double() - b.double()).abs().max() / b.double().abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("batch,L,dm,heads,dk,dv,npred", [
    (1, 128, 64, 1, 64, 64, 0),       # one tile
    (2, 300, 128, 3, 64, 64, 16),     # ragged rows, partial column tile + R
    (1, 257, 192, 2, 128, 64, 32),    # d_k = 128, d_v = 64, npred = 32
    (3, 100, 64, 5, 32, 96, 8),       # odd head widths (multiples of 32)
])
def test_qkv_matches_reference_matmul(batch, L, dm, heads, dk, dv, npred, reference):
    x, wq, wk, wv, pm, w, q, k, v, r = _run(batch, L, dm, heads, dk, dv, npred)
    xs = x.double().numpy()
    for b in range(batch):
        for h in range(heads):
            pr = b * heads + h
            # the reference's own f64 matmul (P/src/linalg.cpp:11-17) of the same bf16 operands
            for got, wl in ((q, wq), (k, wk), (v, wv)):
                want = reference.project(xs[b], wl[h].double().numpy())
                assert _rel(got[pr], torch.from_numpy(want)) <= 1e-2
        if npred:
            want = reference.project(xs[b], pm.to(torch.bfloat16).double().numpy())
            assert _rel(r[b], torch.from_numpy(want)) <= 1e-5


@pytest.mark.parametrize("cfg", ["c2", "c4_slice"])
def test_qkv_full_size_vs_torch(cfg):
    # C2: batch 16, L 4096, d_model 512, 8 heads of 64 (+ k = 16 predictor
    # columns); C4 shape with fewer rows (d_model 1024, 16 heads)
    batch, L, dm, heads = (16, 4096, 512, 8) if cfg == "c2" else (2, 16384, 1024, 16)
    dk = dv = 64
    npred = 16
    x, wq, wk, wv, pm = _inputs(batch, L, dm, heads, dk, dv, npred, seed=11)
    w = ops.pack_qkv_weights(wq, wk, wv, pm).cuda()
    xd = x.cuda()
    q, k, v, r = ops.project_qkv(xd, w, heads, dk, dv, npred)
    y = (xd.reshape(-1, dm).float() @ w.float().t())  # fp32 reference of the same bf16 operands
    HK = heads * dk
    for b in (0, batch - 1):
        rows = slice(b * L, (b + 1) * L)
        for h in (0, heads - 1):
            pr = b * heads + h
            assert _rel(q[pr], y[rows, h * dk:(h + 1) * dk]) <= 1e-2
            assert _rel(k[pr], y[rows, HK + h * dk:HK + (h + 1) * dk]) <= 1e-2
            assert _rel(v[pr], y[rows, 2 * HK + h * dv:2 * HK + (h + 1) * dv]) <= 1e-2
        assert _rel(r[b], y[rows, 2 * HK + heads * dv:]) <= 1e-5
    # every element: bf16 rounding of the fp32 result (half an ulp, plus
    # accumulation-order differences)
    qf = q.float().reshape(batch, heads, L, dk).permute(0, 2, 1, 3).reshape(-1, HK)
    err = (qf - y[:, :HK]).abs()
    assert float((err - (y[:, :HK].abs() * 2 ** -8 + 1e-3)).max()) <= 0.0


def test_qkv_errors():
    x = torch.zeros(1, 64, 96, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(3 * 64, 96, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(Exception):
        ops.project_qkv(x, w, 1, 64, 64)  # d_model % 64 != 0 -> Unsupported
    with pytest.raises(ShapeError):
        ops.project_qkv(torch.zeros(1, 64, 128, dtype=torch.bfloat16, device="cuda"), w, 1, 64, 64)
    with pytest.raises(ParamError):
        ops.project_qkv(x.float(), w, 1, 64, 64)


def _sweep(n=20, seed=2718):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        out.append((int(rng.integers(1, 4)), int(rng.choice([1, 31, 32, 33, 127, 128, 129, 255, 384, int(rng.integers(2, 700))])),
                    int(rng.choice([64, 128, 192, 320, 512])), int(rng.integers(1, 7)), int(rng.choice([32, 64, 96, 128])),
                    int(rng.choice([32, 64, 96, 128])), int(rng.choice([0, 1, 7, 8, 16, 17, 32]))))
    return out


@pytest.mark.parametrize("batch,L,dm,heads,dk,dv,npred", _sweep())
def test_qkv_random_shapes(batch, L, dm, heads, dk, dv, npred):
    """Seeded random (batch, L, d_model, heads, d_k, d_v, npred) incl. L = 1, one
    row past / short of a tile, n_out spanning several 256-column tiles, odd
    predictor widths: every element within half a bf16 ulp (+ fp32 accumulation
    noise) of an fp32 matmul of the same bf16 operands; R within 1e-5."""
    x, wq, wk, wv, pm, w, q, k, v, r = _run(batch, L, dm, heads, dk, dv, npred, seed=11 + L + dm)
    xs = x.float()
    for b in range(batch):
        for h in range(heads):
            pr = b * heads + h
            for got, wl in ((q, wq), (k, wk), (v, wv)):
                want = xs[b] @ wl[h].float()
                tol = want.abs() * 2.0 ** -8 + 1e-5 * want.abs().max()   # half a bf16 ulp is 2^-9 relative
                assert bool(((got[pr].float() - want).abs() <= tol).all()), (b, h)
        if npred:
            want = xs[b] @ pm.to(torch.bfloat16).float()
            assert _rel(r[b], want) <= 1e-5
