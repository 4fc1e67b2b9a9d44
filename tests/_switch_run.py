"""Helper for tests/test_gpu_switches.py (not a test module): runs one small
config through the C-ABI in a FRESH process -- the library reads its
kernel-selection switches (DSA_*) once at load -- and saves levels, masks
and Z of both the phase-by-phase path and dsa_pipeline.

    python tests/_switch_run.py <out.npz> <json: {"preset", "pairs", "pair0", "over"}>
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2110_11299_b200 import load_preset, ops  # noqa: E402


def main():
    out, spec = sys.argv[1], json.loads(sys.argv[2])
    p = load_preset(spec["preset"]).replace(**spec.get("over", {}))
    n = spec["pairs"]
    sub = p.replace(batch=n, heads=1)
    q, k, v, P = ops.generate(sub, pair0=spec.get("pair0", 0), npairs=n)
    dev = torch.device("cuda:0")
    qd, kd, vd, Pd = (t.to(dev) for t in (q, k, v, P))
    lv = ops.predict(sub, qd, kd, Pd)
    mask = ops.select(sub, lv)
    z = ops.sparse_attention(sub, qd, kd, vd, mask)
    pipe = ops.Pipeline(sub, device=dev, keep_mask=True)
    zp = pipe(qd, kd, vd, Pd)
    torch.cuda.synchronize()
    rows = ops.mask_rows(sub, mask, n)
    prow = ops.mask_rows(sub, pipe.mask, n)
    rp, cols = ops.to_csr([r for pr in rows for r in pr])
    prp, pcols = ops.to_csr([r for pr in prow for r in pr])
    np.savez(out, lq=ops.levels_rows(lv.lq).float().cpu().numpy(), lk=ops.levels_rows(lv.lk).float().cpu().numpy(),
             sq=lv.sq.cpu().numpy(), sk=lv.sk.cpu().numpy(), rp=rp, cols=cols, prp=prp, pcols=pcols,
             z=z.float().cpu().numpy(), zp=zp.float().cpu().numpy(),
             launches=np.int64(ops.launch_counter()))


if __name__ == "__main__":
    main()
