"""Times each phase of the hot path with CUDA events: every phase is
enqueued `reps` times back to back between two events, so host launch
overhead is hidden behind GPU work (device time per launch)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2110_11299_b200 import load_preset, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_vector")
ap.add_argument("--pairs", type=int, default=0)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
p = load_preset(a.config)
n = a.pairs or p.pairs
sub = p.replace(batch=n, heads=1) if a.pairs else p
q, k, v, P = ops.generate(sub, npairs=n)
qd, kd, vd, Pd = (t.cuda() for t in (q, k, v, P))
ph = ops.Phases(sub, n)
z = torch.empty_like(qd)
fns = {"predict": lambda: ph.predict(qd, kd, Pd), "select": ph.select,
       "attention": lambda: ph.attend(qd, kd, vd, z)}
for f in fns.values():  # warm up in pipeline order
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
for name, f in fns.items():
    f()
    e0.record()
    for _ in range(a.reps):
        f()
    e1.record()
    e1.synchronize()
    res[name] = round(e0.elapsed_time(e1) / a.reps, 4)
res["total"] = round(sum(res.values()), 4)
print(a.config, res, flush=True)
