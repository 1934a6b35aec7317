"""K6 experiment: time one 4-way pass (k6_quad.cuh) on 2^28 int32 keys = groups
of four sorted runs of L, with the 4-way co-rank tiles computed by torch's
stable sort (a stand-in for a partition kernel, not timed), checked against
torch.sort, vs two 2-way levels of the fused K3 (measured: the K3 launch of a
sort whose input is already runs of L: msort on runs via the segmented call is
not that, so the reference is the bench's per-level K3 time).

    python scripts/k6_experiment.py [--log2n 28] [--log2L 24]
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import msort_inputs as mi  # noqa: E402
import paper_2211_16479_b200 as ms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=28)
ap.add_argument("--log2L", type=int, default=24)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
n, L = 1 << a.log2n, 1 << a.log2L
Tm = 126 * 68
keys = mi.keys_torch(n, 4, "u31", device="cuda")
# runs of L: sort each segment
off = torch.arange(0, n + 1, L, dtype=torch.int64, device="cuda")
ms.msort_sort_segmented(keys, off)
torch.cuda.synchronize()
tiles = []
expect = torch.empty_like(keys)
G = 4 * L
for g in range(n // G):
    grp = keys[g * G:(g + 1) * G]
    sv, si = torch.sort(grp, stable=True)
    expect[g * G:(g + 1) * G] = sv
    run = (si // L).to(torch.int8)
    cnt = torch.stack([(run == r).to(torch.int32).cumsum(0) for r in range(4)], 1)  # [G, 4]
    d = torch.arange(0, G, Tm, device="cuda")
    s0 = torch.zeros(d.numel(), 4, dtype=torch.int64, device="cuda")
    s0[1:] = cnt[d[1:] - 1].to(torch.int64)
    s1 = torch.empty_like(s0)
    s1[:-1] = s0[1:]
    s1[-1] = torch.tensor([L, L, L, L], device="cuda")
    t = torch.empty(d.numel(), 9, dtype=torch.int64, device="cuda")
    t[:, 0] = g * G + d
    for r in range(4):
        t[:, 1 + r] = g * G + r * L + s0[:, r]
        t[:, 5 + r] = s1[:, r] - s0[:, r]
    tiles.append(t)
    del sv, si, run, cnt
tiles = torch.cat(tiles).contiguous()
nt = tiles.shape[0]
dst = torch.empty_like(keys)
f = ms.lib.msort_debug_k6_pass
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
s = torch.cuda.current_stream().cuda_stream
rc = f(keys.data_ptr(), dst.data_ptr(), tiles.data_ptr(), nt, s)
torch.cuda.synchronize()
ok = bool(torch.equal(dst, expect))
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f(keys.data_ptr(), dst.data_ptr(), tiles.data_ptr(), nt, s)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
med = statistics.median(ts)
print(json.dumps({"n": n, "L": L, "tiles": nt, "rc": rc, "correct": ok, "ms": round(med, 4),
                  "gbs": round(2 * n * 4 / med / 1e6, 1)}), flush=True)
