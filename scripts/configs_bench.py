"""Time every BASELINE.json config on one GPU (out of place, workspace preallocated).

    python scripts/configs_bench.py [--reps 10]
C1 2^16 int32 u31 | C2 2^24 int32 (random / sorted / reversed) | C3 2^26 int64 mod 1000 + uint32
index payload | C4 2^27 uint32 + uint32 index payload | C5 2^28 int32 (one shard).
One JSON line per config: median ms (CUDA events), G keys/s, GB/s of one read + one write.
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
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()

CFG = [("C1", 16, 0, "u31", False, None), ("C2", 24, 1, "u31", False, None),
       ("C2s", 24, 1, "u31", False, "sorted"), ("C2r", 24, 1, "u31", False, "reversed"),
       ("C3", 26, 2, ("mod", 1000), True, None), ("C4", 27, 3, "u32", True, None),
       ("C5", 28, 4, "u31", False, None)]
for name, lg, seed, dist, pairs, variant in CFG:
    n = 1 << lg
    kin = mi.keys_torch(n, seed, dist, device="cuda")
    if variant:
        kin = torch.sort(kin.to(torch.int64))[0].to(kin.dtype)
        if variant == "reversed":
            kin = kin.flip(0).contiguous()
    kout = torch.empty_like(kin)
    vin = torch.arange(n, dtype=torch.int32, device="cuda") if pairs else None
    vout = torch.empty_like(vin) if pairs else None
    ws = ms.workspace(n, kin.dtype, pairs, device="cuda")
    for _ in range(3):
        ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
    torch.cuda.synchronize()
    ts = []
    ms.profile_reset()
    ms.profile_enable(True)
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    med = statistics.median(ts)
    ms.profile_enable(False)
    prof = {k: round(v[1] / a.reps, 4) for k, v in ms.profile_read().items() if v[0]}
    rec = kin.element_size() + (4 if pairs else 0)
    print(json.dumps({"config": name, "n": n, "pairs": pairs, "ms": round(med, 4),
                      "gkeys_s": round(n / med / 1e6, 3),
                      "one_pass_gbs": round(2 * n * rec / med / 1e6, 1), "phase_ms": prof}), flush=True)
