"""Does the selection of one pair chunk overlap the attention of another?
Two independent pair sets A and B of one config: select(A) on stream 1 and
attention(B) on stream 2, alone and together (CUDA events around both).
The selection kernels are issue-bound and the attention gather-bound, so
together < alone + alone means chunk pipelining inside dsa_pipeline pays."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2110_11299_b200 import load_preset, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4_threshold")
ap.add_argument("--pairs", type=int, default=32)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
p = load_preset(a.config)
n = a.pairs
sub = p.replace(batch=n, heads=1)
sets = []
for i in range(2):
    q, k, v, P = ops.generate(sub, pair0=i * n, npairs=n)
    qd, kd, vd, Pd = (t.cuda() for t in (q, k, v, P))
    ph = ops.Phases(sub, n)
    z = torch.empty_like(qd)
    ph.predict(qd, kd, Pd)
    ph.select()
    ph.attend(qd, kd, vd, z)
    sets.append((ph, qd, kd, vd, z))
torch.cuda.synchronize()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
A, B = sets


def run(sel: bool, att: bool) -> float:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    torch.cuda.synchronize()
    e0.record()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    for _ in range(a.reps):
        if sel:
            A[0].select(stream=s1)
        if att:
            B[0].attend(B[1], B[2], B[3], B[4], stream=s2)
    cur.wait_stream(s1)
    cur.wait_stream(s2)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / a.reps


for _ in range(2):
    ts, ta, tb = run(True, False), run(False, True), run(True, True)
    print(f"{a.config} pairs={n}: select {ts:.3f} ms, attention {ta:.3f} ms, both {tb:.3f} ms "
          f"(sum {ts + ta:.3f}, overlap gain {(ts + ta) / tb:.3f}x)", flush=True)
