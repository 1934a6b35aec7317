"""Sort latency per size (keys only, int32 u31, out-of-place, workspace preallocated).

    python scripts/latency.py [--sizes 16,20,24,26,28] [--reps 50]
Prints one JSON line per size: ms (median of reps, CUDA events), G keys/s, launches.
"""
import argparse
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
ap.add_argument("--sizes", default="16,18,20,22,24,26,28")
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
for lg in [int(x) for x in a.sizes.split(",")]:
    n = 1 << lg
    kin = mi.keys_torch(n, 0, "u31", device="cuda")
    kout = torch.empty_like(kin)
    ws = ms.workspace(n, kin.dtype, False, device="cuda")
    for _ in range(5):
        ms.msort_sort_out(kin, kout, ws=ws)
    torch.cuda.synchronize()
    ts = []
    l0 = ms.launch_count()
    ms.profile_reset()
    ms.profile_enable(True)
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ms.msort_sort_out(kin, kout, ws=ws)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    launches = (ms.launch_count() - l0) / a.reps
    ms.profile_enable(False)
    prof = {k: round(v[1] / a.reps, 4) for k, v in ms.profile_read().items() if v[0]}
    med = statistics.median(ts)
    ok = bool((kout[1:] >= kout[:-1]).all())
    print(json.dumps({"log2n": lg, "ms": round(med, 4), "min_ms": round(min(ts), 4),
                      "gkeys_s": round(n / med / 1e6, 3), "launches": launches, "phase_ms": prof, "sorted": ok}))
