"""Host<->device copy ceilings for the e2e leg: 1 GiB pinned H2D alone, D2H
alone, both directions at once on two streams (full duplex?), each timed on
the device with CUDA events.  Prints one JSON line."""
import json

import torch

n = 1 << 28
dev = torch.device("cuda:0")
h_in = torch.empty(n, dtype=torch.int32).pin_memory()
h_out = torch.empty(n, dtype=torch.int32).pin_memory()
d_a = torch.empty(n, dtype=torch.int32, device=dev)
d_b = torch.empty(n, dtype=torch.int32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
gb = n * 4 / 1e9


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    for _ in range(reps):
        fn()
    f1, f2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f1.record(s1)
    f2.record(s2)
    torch.cuda.synchronize()
    return max(e0.elapsed_time(f1), e0.elapsed_time(f2)) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


r = {}
r["h2d_ms"] = timed(h2d)
r["d2h_ms"] = timed(d2h)
r["both_ms"] = timed(both)
r["h2d_gbs"] = gb / r["h2d_ms"] * 1e3
r["d2h_gbs"] = gb / r["d2h_ms"] * 1e3
r["both_gbs_each"] = gb / r["both_ms"] * 1e3
print(json.dumps(r))
