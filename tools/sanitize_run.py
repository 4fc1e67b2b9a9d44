"""One small invocation of every kernel family (each BASELINE config's mask
mode at reduced L, phases + dsa_pipeline, the QKV GEMM) for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2110_11299_b200 import load_preset, ops  # noqa: E402

CASES = [("c0_smoke", {}), ("c1_bert_base", {"L": 512, "keep": 26}), ("c2_vector", {"L": 1024, "keep": 51}),
         ("c3_block", {"L": 1024, "keep": 5}), ("c4_threshold", {"L": 1024, "cap": 50})]
for name, over in CASES:
    p = load_preset(name).replace(**over)
    sub = p.replace(batch=2, heads=1)
    q, k, v, P = ops.generate(sub, npairs=2)
    qd, kd, vd, Pd = (t.cuda() for t in (q, k, v, P))
    lv = ops.predict(sub, qd, kd, Pd)
    m = ops.select(sub, lv)
    z = ops.sparse_attention(sub, qd, kd, vd, m)
    zp = ops.Pipeline(sub, keep_mask=True)(qd, kd, vd, Pd)
    torch.cuda.synchronize()
    print(name, "ok", float(z.float().abs().sum()), float(zp.float().abs().sum()))
x = torch.randn(1, 256, 128, device="cuda").to(torch.bfloat16)
w = (torch.randn(2 * (64 + 64 + 64) + 16, 128, device="cuda") / 11).to(torch.bfloat16)
ops.project_qkv(x, w, 2, 64, 64, 16)
torch.cuda.synchronize()
print("qkv ok")
