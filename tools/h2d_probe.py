"""H2D / D2H bandwidth probe: one pinned 201 MB copy on one stream vs the
same bytes split over 2 or 3 streams (copy engines), plus concurrent D2H."""
import torch

dev = torch.device("cuda:0")
n = 201330688 // 2
h = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
d = torch.empty(n, dtype=torch.bfloat16, device=dev)
zo = torch.empty(67108864 // 2, dtype=torch.bfloat16, pin_memory=True)
zd = torch.empty(67108864 // 2, dtype=torch.bfloat16, device=dev)
streams = [torch.cuda.Stream(device=dev) for _ in range(4)]


def run(parts, with_d2h, reps=5):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        chunk = n // parts
        for p in range(parts):
            s = streams[p]
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[p * chunk:(p + 1) * chunk].copy_(h[p * chunk:(p + 1) * chunk], non_blocking=True)
        if with_d2h:
            s = streams[3]
            s.wait_event(e0)
            with torch.cuda.stream(s):
                zo.copy_(zd, non_blocking=True)
    for s in streams:
        e1.wait(s) if False else torch.cuda.current_stream().wait_stream(s)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"parts={parts} d2h={with_d2h}: {ms:.3f} ms per 201 MB -> {2 * n / ms / 1e6:.1f} GB/s H2D")


for parts in (1, 2, 3):
    for dd in (False, True):
        run(parts, dd)
