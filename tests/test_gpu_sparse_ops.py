"""The reference's unfused sparse operators on the device (dsa_sddmm_f64,
dsa_sparse_softmax_f64, dsa_spmm_f64; P/src/sparse.cpp:38-91) through the
C ABI: against a float64 numpy restatement on ragged CSR masks (empty rows,
single-entry rows, full rows), and their chain against the fused
dsa_sparse_attention.  (Bit-identity with the reference's scalar kernels is
checked in tests/cpp/test_shim.cpp, linked with the reference.)"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ragged_csr(rng, L, max_keep):
    rows = []
    for i in range(L):
        n = int(rng.integers(0, max_keep + 1))
        if i == 3:
            n = 0
        if i == 5:
            n = 1
        if i == 7:
            n = L
        rows.append(np.sort(rng.choice(L, size=n, replace=False)).astype(np.uint32))
    rowptr = np.zeros(L + 1, dtype=np.uint64)
    rowptr[1:] = np.cumsum([len(r) for r in rows])
    return rows, rowptr, np.concatenate(rows).astype(np.uint32)


@pytest.mark.parametrize("L,d,dv,scale", [(200, 64, 64, True), (97, 24, 40, False), (512, 128, 128, True)])
def test_unfused_operators_match_float64_reference(L, d, dv, scale):
    import torch
    from paper_2110_11299_b200 import ops

    rng = np.random.default_rng(L + d)
    q, k, v = rng.standard_normal((L, d)), rng.standard_normal((L, d)), rng.standard_normal((L, dv))
    rows, rowptr, cols = _ragged_csr(rng, L, 40)
    dev = "cuda"
    qd, kd, vd = (torch.from_numpy(x).to(dev) for x in (q, k, v))
    rp = torch.from_numpy(rowptr.view(np.int64)).to(dev)
    cl = torch.from_numpy(cols.view(np.int32)).to(dev)

    s = ops.sddmm(qd, kd, rp, cl, scale)
    sc = 1.0 / np.sqrt(d) if scale else 1.0
    s_ref = np.concatenate([(k[r.astype(np.int64)] @ q[i]) * sc for i, r in enumerate(rows)])
    assert np.abs(s.cpu().numpy() - s_ref).max() <= 1e-13 * np.abs(s_ref).max()

    w, empty = ops.sparse_softmax(s, rp)
    wn, en = w.cpu().numpy(), empty.cpu().numpy()
    sn = s.cpu().numpy()
    for i, r in enumerate(rows):
        b, e = int(rowptr[i]), int(rowptr[i + 1])
        assert en[i] == (1 if b == e else 0)
        if b == e:
            continue
        x = np.exp(sn[b:e] - sn[b:e].max())
        assert np.abs(wn[b:e] - x / x.sum()).max() <= 1e-15
    assert wn[int(rowptr[5])] == 1.0

    z = ops.spmm(w, rp, cl, vd).cpu().numpy()
    z_ref = np.stack([wn[int(rowptr[i]):int(rowptr[i + 1])] @ v[r.astype(np.int64)] if len(r) else np.zeros(dv)
                      for i, r in enumerate(rows)])
    assert np.abs(z - z_ref).max() <= 1e-13 * max(1.0, np.abs(z_ref).max())
    assert not z[3].any()


def test_unfused_chain_equals_fused_attention():
    """sddmm -> sparse_softmax -> spmm on C0's mask == dsa_sparse_attention (f32 bar)."""
    import torch
    from paper_2110_11299_b200 import load_preset, ops

    p = load_preset("c0_smoke")
    q, k, v, P = ops.generate(p)
    qd, kd, vd, Pd = (t.cuda() for t in (q, k, v, P))
    mask = ops.select(p, ops.predict(p, qd, kd, Pd))
    z = ops.sparse_attention(p, qd, kd, vd, mask)[0].double()
    cols = mask.cols[: p.L * p.keep].contiguous()
    rp = torch.arange(0, p.L * p.keep + 1, p.keep, dtype=torch.int64, device="cuda")
    cl = cols.view(torch.int32) if cols.dtype != torch.int32 else cols
    s = ops.sddmm(qd[0].double().contiguous(), kd[0].double().contiguous(), rp, cl, True)
    w, empty = ops.sparse_softmax(s, rp)
    zc = ops.spmm(w, rp, cl, vd[0].double().contiguous())
    assert not empty.any()
    assert ((zc - z).abs().max() / z.abs().max()).item() <= 1e-5


def test_unfused_operator_errors():
    import torch
    from paper_2110_11299_b200 import ops
    from paper_2110_11299_b200.errors import ParamError, ShapeError

    q = torch.zeros((4, 8), dtype=torch.float64, device="cuda")
    rp = torch.zeros(5, dtype=torch.int64, device="cuda")
    cl = torch.zeros(0, dtype=torch.int32, device="cuda")
    assert ops.sddmm(q, q, rp, cl).numel() == 0
    with pytest.raises(ShapeError):
        ops.sddmm(q, torch.zeros((4, 9), dtype=torch.float64, device="cuda"), rp, cl)
    with pytest.raises(ParamError):
        ops.sddmm(q.float(), q.float(), rp, cl)
    w, e = ops.sparse_softmax(torch.zeros(0, dtype=torch.float64, device="cuda"), rp)
    assert e.cpu().tolist() == [1, 1, 1, 1]
    with pytest.raises(ShapeError):
        ops.spmm(w, rp, cl, torch.zeros((5, 8), dtype=torch.float64, device="cuda"))
    assert not ops.spmm(w, rp, cl, q).any()


@pytest.mark.parametrize("rows,cols,keep", [(1, 1, 1), (37, 91, 7), (64, 2048, 102), (5, 25600, 300), (9, 513, 513)])
def test_row_topk_f64_matches_reference_rule(rows, cols, keep):
    """dsa_row_topk_f64 == row_topk_indices (P/src/linalg.cpp:69-85): value desc,
    lowest column among equals, ascending output; heavy ties, -0 == +0."""
    import torch
    from paper_2110_11299_b200 import ops
    from paper_2110_11299_b200.errors import ParamError

    rng = np.random.default_rng(rows * cols)
    s = np.floor(rng.standard_normal((rows, cols)) * 1.5)     # a handful of distinct values: ties everywhere
    s[0, : min(4, cols)] = [-0.0, 0.0, -0.0, 0.0][: min(4, cols)]
    got = ops.row_topk(torch.from_numpy(s).cuda(), keep).cpu().numpy()
    order = np.argsort(-s, axis=1, kind="stable")[:, :keep]   # stable: the lowest column first among equals
    assert np.array_equal(got, np.sort(order, axis=1))
    with pytest.raises(ParamError):
        ops.row_topk(torch.from_numpy(s).cuda(), cols + 1)
    with pytest.raises(ParamError):
        ops.row_topk(torch.from_numpy(s).cuda(), 0)
