"""Times each phase of the hot path with CUDA events (median of N)."""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2110_11299_b200 import load_preset, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_vector")
ap.add_argument("--pairs", type=int, default=0)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
p = load_preset(a.config)
n = a.pairs or p.pairs
sub = p.replace(batch=n, heads=1) if a.pairs else p
q, k, v, P = ops.generate(sub, npairs=n)
qd, kd, vd, Pd = (t.cuda() for t in (q, k, v, P))
ph = ops.Phases(sub, n)
z = torch.empty_like(qd)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
res = {"predict": [], "select": [], "attention": []}
for i in range(a.reps + 2):
    ev[0].record()
    ph.predict(qd, kd, Pd)
    ev[1].record()
    ph.select()
    ev[2].record()
    ph.attend(qd, kd, vd, z)
    ev[3].record()
    ev[3].synchronize()
    if i >= 2:
        res["predict"].append(ev[0].elapsed_time(ev[1]))
        res["select"].append(ev[1].elapsed_time(ev[2]))
        res["attention"].append(ev[2].elapsed_time(ev[3]))
print(a.config, {k_: round(statistics.median(v_), 4) for k_, v_ in res.items()}, flush=True)
