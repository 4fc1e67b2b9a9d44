import sys, torch
sys.path.insert(0, '.')
from paper_2110_11299_b200 import load_preset, ops
for name in ["c2_vector", "c4_threshold"]:
    p = load_preset(name)
    n = 128 if name == "c2_vector" else 64
    sub = p.replace(batch=n, heads=1)
    q, k, v, P = ops.generate(sub, npairs=n)
    qd, kd, Pd = q.cuda(), k.cuda(), P.cuda()
    ph = ops.Phases(sub, n)
    ph.predict(qd, kd, Pd)
    torch.cuda.synchronize()
    # plan: [x64 | xhat | ...]; x64 empty for the tc path -> xhat at offset 0
    ws = ph.ws
    L, KD = sub.L, sub.k
    off_floats = n * 2 * L * (KD + 1)
    cnt = ws[off_floats * 4: off_floats * 4 + 8].view(torch.int64).item()
    print(name, "deferred levels", cnt, "of", n * 2 * L * KD, "(%.4f%%)" % (100.0 * cnt / (n * 2 * L * KD)))
