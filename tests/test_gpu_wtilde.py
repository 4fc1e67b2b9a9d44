"""The reference's own predictor entry point on the GPU: approx_scores /
approx_scores_from_r with the trainable per-head k x k W~
(P/src/predictor.cpp:67-80, P/src/trainer.cpp:162,173-175) through
dsa_predict_wtilde, against the reference implementation itself
(oracle/_ref): R = matmul(X, P), levels/scale of quantize(matmul(R, W~)).

* R, levels and scales: bit-exact (f64 and f32 Matrices, INT4 / INT8 / 2-bit,
  k 16 / 32, per-tensor; per-row scope against quantize() of each row);
* the row top-k mask selected from those levels (dsa_select) equals
  predicted_topk_mask on the exact-integer S~."""
import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import load_preset, ops

pytestmark = pytest.mark.gpu


def _inputs(batch, heads, L, dm, k, f32, seed, reference):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(batch, L, dm))
    P = reference.init_projection(dm, k, seed)  # the reference's ternary projection
    wq = rng.normal(scale=0.3, size=(heads, k, k))
    wk = rng.normal(scale=0.3, size=(heads, k, k))
    if f32:
        x, wq, wk = (a.astype(np.float32).astype(np.float64) for a in (x, wq, wk))
        P = P.astype(np.float32).astype(np.float64)
    return x, P, wq, wk


@pytest.mark.parametrize("batch,heads,L,dm,k,bits,f32", [
    (2, 3, 257, 64, 16, 4, False),
    (1, 2, 512, 128, 32, 8, False),
    (2, 2, 300, 96, 16, 2, True),
    (1, 4, 1024, 512, 16, 4, False),
])
def test_wtilde_levels_match_reference(batch, heads, L, dm, k, bits, f32, reference):
    x, P, wq, wk = _inputs(batch, heads, L, dm, k, f32, 100 + L, reference)
    p = load_preset("c0_smoke").replace(batch=batch, heads=heads, L=L, k=k, bits=bits,
                                        round_proj_f32=f32, d=64, keep=min(13, L))
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    lv, r = ops.predict_wtilde(p, t(wq), t(wk), x=t(x), P=t(P))
    torch.cuda.synchronize()
    glq = ops.levels_rows(lv.lq).float().cpu().numpy().astype(np.int32)
    glk = ops.levels_rows(lv.lk).float().cpu().numpy().astype(np.int32)
    rg = r.cpu().numpy()
    for b in range(batch):
        for h in range(heads):
            pr = b * heads + h
            lq, sq, rr = reference.levels_wtilde(wq[h], bits, f32, x=x[b], p=P)
            lk, sk, _ = reference.levels_wtilde(wk[h], bits, f32, x=x[b], p=P)
            assert np.array_equal(rg[b], rr), "R = X P differs"
            assert np.array_equal(glq[pr], lq) and np.array_equal(glk[pr], lk), (b, h)
            assert lv.sq[pr].item() == sq and lv.sk[pr].item() == sk
    # the R input path (approx_scores_from_r) gives the same levels
    lv2, _ = ops.predict_wtilde(p, t(wq), t(wk), r=r)
    torch.cuda.synchronize()
    assert torch.equal(lv2.lq, lv.lq) and torch.equal(lv2.lk, lv.lk) and torch.equal(lv2.sq, lv.sq)


def test_wtilde_mask_matches_reference_topk(reference, oracle):
    batch, heads, L, dm, k = 1, 2, 640, 64, 16
    x, P, wq, wk = _inputs(batch, heads, L, dm, k, False, 7, reference)
    p = load_preset("c0_smoke").replace(batch=batch, heads=heads, L=L, k=k, bits=4, dtype="bf16",
                                        round_proj_f32=False, keep=37)
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    lv, _ = ops.predict_wtilde(p, t(wq), t(wk), x=t(x), P=t(P))
    mask = ops.select(p, lv)
    torch.cuda.synchronize()
    cols = mask.cols[: heads * L * p.keep].cpu().numpy().astype(np.uint32).reshape(heads, L, p.keep)
    for h in range(heads):
        lq, _, _ = reference.levels_wtilde(wq[h], 4, x=x[0], p=P)
        lk, _, _ = reference.levels_wtilde(wk[h], 4, x=x[0], p=P)
        S = oracle.scores_int(lq, lk).astype(np.float64)
        assert np.array_equal(cols[h], reference.topk_mask(S, p.keep))


def test_wtilde_per_row_scope(reference):
    batch, heads, L, dm, k = 1, 1, 200, 64, 16
    x, P, wq, wk = _inputs(batch, heads, L, dm, k, False, 9, reference)
    p = load_preset("c1_bert_base").replace(batch=batch, heads=heads, L=L, k=k, keep=10)
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    lv, r = ops.predict_wtilde(p, t(wq), t(wk), x=t(x), P=t(P))
    torch.cuda.synchronize()
    glq = ops.levels_rows(lv.lq)[0].float().cpu().numpy().astype(np.int32)
    _, _, rr = reference.levels_wtilde(wq[0], 4, x=x[0], p=P)
    for i in range(L):  # per-row scope: quantize() of each 1 x k row of R W~
        lvr, s, _ = reference.levels_wtilde(wq[0], 4, r=rr[i:i + 1])
        assert np.array_equal(glq[i], lvr[0]) and lv.sq[0, i].item() == s


def _sweep(n=16, seed=31337):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        out.append((int(rng.integers(1, 4)), int(rng.integers(1, 5)), int(rng.choice([1, 31, 64, 129, 255, 777, int(rng.integers(2, 900))])),
                    int(rng.choice([16, 32, 48, 64, 100, 256])), int(rng.choice([16, 32])), int(rng.choice([2, 4, 8])),
                    bool(rng.random() < 0.5)))
    return [c for c in out if c[4] <= c[3]]


@pytest.mark.parametrize("batch,heads,L,dm,k,bits,f32", _sweep())
def test_wtilde_random_shapes(batch, heads, L, dm, k, bits, f32, reference):
    """Seeded random (batch, heads, L, d_model, k, bits, precision): R, levels and
    scales bit-exact against the reference library, degenerate L = 1 included."""
    x, P, wq, wk = _inputs(batch, heads, L, dm, k, f32, 5 * L + dm + bits, reference)
    p = load_preset("c0_smoke").replace(batch=batch, heads=heads, L=L, k=k, bits=bits,
                                        round_proj_f32=f32, d=64, keep=1)
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    lv, r = ops.predict_wtilde(p, t(wq), t(wk), x=t(x), P=t(P))
    torch.cuda.synchronize()
    glq = ops.levels_rows(lv.lq).float().cpu().numpy().astype(np.int32)
    glk = ops.levels_rows(lv.lk).float().cpu().numpy().astype(np.int32)
    rg = r.cpu().numpy()
    for b in range(batch):
        for h in range(heads):
            pr = b * heads + h
            lq, sq, rr = reference.levels_wtilde(wq[h], bits, f32, x=x[b], p=P)
            lk, sk, _ = reference.levels_wtilde(wk[h], bits, f32, x=x[b], p=P)
            assert np.array_equal(rg[b], rr), "R = X P differs"
            assert np.array_equal(glq[pr], lq) and np.array_equal(glk[pr], lk), (b, h)
            assert lv.sq[pr].item() == sq and lv.sk[pr].item() == sk
