"""Runs the hot path once per phase on a BASELINE config (for ncu captures)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2110_11299_b200 import load_preset, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_vector")
ap.add_argument("--pairs", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--pipeline", action="store_true", help="dsa_pipeline (fused kernels) instead of the phases")
a = ap.parse_args()
p = load_preset(a.config)
n = a.pairs or p.pairs
sub = p.replace(batch=n, heads=1) if a.pairs else p
q, k, v, P = ops.generate(sub, npairs=n)
qd, kd, vd, Pd = (t.cuda() for t in (q, k, v, P))
ph = ops.Phases(sub, n)
z = torch.empty_like(qd)
pipe = ops.Pipeline(sub, pairs=n)
for _ in range(a.reps):
    if a.pipeline:
        pipe(qd, kd, vd, Pd, out=z)
        continue
    ph.predict(qd, kd, Pd)
    ph.select()
    ph.attend(qd, kd, vd, z)
torch.cuda.synchronize()
print("ok", float(z.float().abs().sum()))
