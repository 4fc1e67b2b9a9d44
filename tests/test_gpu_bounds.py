"""Out-of-bounds write checks (compute-sanitizer is closed on this GPU pool,
profiles/r02_sanitizer_unavailable.log): every buffer the C-ABI writes --
levels, scales, mask lists / CSR, empty-row flags, Z, and the caller
workspace -- sits between 4 KB guard bands of a known byte pattern; after
predict -> select -> attention and after dsa_pipeline the guards must be
intact and every output byte written where the contract says so.  Ragged
shapes (L not a multiple of any tile) are included."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import _abi, load_preset, ops

pytestmark = pytest.mark.gpu

GUARD = 4096
PAT = 0xA5


class Guarded:
    def __init__(self, nbytes, dev):
        self.n = max(int(nbytes), 1)
        self.buf = torch.full((self.n + 2 * GUARD,), PAT, dtype=torch.uint8, device=dev)

    @property
    def ptr(self):
        return self.buf.data_ptr() + GUARD

    def intact(self):
        b = self.buf.cpu().numpy()
        return bool((b[:GUARD] == PAT).all() and (b[GUARD + self.n:] == PAT).all())


CASES = [("c0_smoke", {"L": 333, "keep": 17}), ("c1_bert_base", {"L": 1000, "keep": 51}),
         ("c2_vector", {"L": 1004, "keep": 51}), ("c2_vector", {"L": 4096, "keep": 205}),
         ("c3_block", {"L": 1000, "keep": 5}), ("c3_block", {"L": 2048, "keep": 7}),
         ("c4_threshold", {"L": 1500, "cap": 60}), ("c4_threshold", {"L": 700, "cap": 9})]


@pytest.mark.parametrize("name,over", CASES)
def test_outputs_stay_in_bounds(name, over):
    p = load_preset(name).replace(**over)
    pairs = 3
    sub = p.replace(batch=pairs, heads=1)
    dev = torch.device("cuda:0")
    q, k, v, P = ops.generate(sub, npairs=pairs)
    qd, kd, vd, Pd = (t.to(dev) for t in (q, k, v, P))
    c = ops.config_of(sub)
    lib = _abi.lib()
    esz = 2 if sub.dtype == "bf16" else 4
    nsc = pairs if sub.quant_scope == "tensor" else pairs * sub.L
    ws = Guarded(lib.dsa_workspace_bytes(C.byref(c)), dev)
    lq, lk = (Guarded(pairs * sub.L * sub.k * 2, dev) for _ in range(2))
    sq, sk = (Guarded(nsc * 8, dev) for _ in range(2))
    cap = lib.dsa_mask_capacity(C.byref(c))
    cols = Guarded(cap * 4, dev)
    rp = Guarded((pairs * sub.L + 1) * 8, dev) if sub.mask_mode == "threshold" else None
    er = Guarded(pairs * sub.L, dev)
    z = Guarded(pairs * sub.L * sub.d * esz, dev)
    st = torch.cuda.current_stream().cuda_stream
    _abi.check(lib.dsa_predict(C.byref(c), qd.data_ptr(), kd.data_ptr(), Pd.data_ptr(), lq.ptr, lk.ptr, sq.ptr,
                               sk.ptr, ws.ptr, ws.n, st))
    m = _abi.DsaMask()
    m.cols, m.rowptr, m.capacity, m.empty_rows = cols.ptr, rp.ptr if rp else None, cap, er.ptr
    _abi.check(lib.dsa_select(C.byref(c), lq.ptr, lk.ptr, sq.ptr, sk.ptr, C.byref(m), ws.ptr, ws.n, st))
    _abi.check(lib.dsa_sparse_attention(C.byref(c), qd.data_ptr(), kd.data_ptr(), vd.data_ptr(), C.byref(m), z.ptr,
                                        st))
    torch.cuda.synchronize()
    bufs = {"workspace": ws, "levels_q": lq, "levels_k": lk, "scale_q": sq, "scale_k": sk, "cols": cols,
            "empty_rows": er, "z": z}
    if rp:
        bufs["rowptr"] = rp
    for nm, b in bufs.items():
        assert b.intact(), f"{name}: write outside {nm}"
    zz = z.buf[GUARD:GUARD + z.n].cpu().numpy()
    assert not (zz == PAT).all(), "Z not written"
    # the fused / chunked pipeline into fresh guarded buffers
    ws2 = Guarded(lib.dsa_workspace_bytes(C.byref(c)), dev)
    z2 = Guarded(pairs * sub.L * sub.d * esz, dev)
    cols2 = Guarded(cap * 4, dev)
    rp2 = Guarded((pairs * sub.L + 1) * 8, dev) if sub.mask_mode == "threshold" else None
    m2 = _abi.DsaMask()
    m2.cols, m2.rowptr, m2.capacity, m2.empty_rows = cols2.ptr, rp2.ptr if rp2 else None, cap, None
    _abi.check(lib.dsa_pipeline(C.byref(c), qd.data_ptr(), kd.data_ptr(), vd.data_ptr(), Pd.data_ptr(), z2.ptr,
                                C.byref(m2), ws2.ptr, ws2.n, st))
    torch.cuda.synchronize()
    for nm, b in {"pipeline workspace": ws2, "pipeline z": z2, "pipeline cols": cols2}.items():
        assert b.intact(), f"{name}: write outside {nm}"
    assert np.array_equal(z2.buf[GUARD:GUARD + z2.n].cpu().numpy(), zz) or sub.mask_mode == "colvec"
