"""Runs a BASELINE config on the GPU and writes reference fixtures for some
(b,h) pairs: the predicted mask (DSAMASK, P/src/mask.cpp:75-89) and the
attention output Z (DSAC, P/src/serialize.cpp:38-63), readable by the
reference tools (e.g. `dataflow --config {masks:[...]}` consumes mask files,
P/src/cli_commands.cpp:394-399).

usage: python tools/export_fixtures.py --config c2_vector --pairs 0 5 --out golden_out
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2110_11299_b200 import fixtures, load_preset, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2_vector")
ap.add_argument("--pairs", type=int, nargs="+", default=[0])
ap.add_argument("--out", default="golden_out")
a = ap.parse_args()
p = load_preset(a.config)
n = max(a.pairs) + 1
sub = p.replace(batch=n, heads=1)
q, k, v, P = ops.generate(sub, npairs=n)
dev = torch.device("cuda:0")
qd, kd, vd, Pd = (t.to(dev) for t in (q, k, v, P))
lv = ops.predict(sub, qd, kd, Pd)
mask = ops.select(sub, lv)
z = ops.sparse_attention(sub, qd, kd, vd, mask)
torch.cuda.synchronize()
for pr in a.pairs:
    print(fixtures.export_pair(sub, mask, z, pr, a.out))
