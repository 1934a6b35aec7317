"""Batched (segmented) sort timings on one GPU.

    python scripts/segmented_bench.py [--reps 20]

Workloads: 2^24 int32 keys (uniform [0, 2^31), counter-mode SplitMix64 seed 1)
cut into segments of a fixed length L (or uniform random lengths 1..L, seed 9),
keys only and with a uint32 index payload.  One JSON line per workload: median
ms (CUDA events around msort_sort_segmented, segment table upload included;
host_enqueue_ms = the call's own host time, binning and staging included),
G keys/s, and the HBM roofline fraction of one read + one write of every
record (the floor for segments that fit one CTA).
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import msort_inputs as mi  # noqa: E402
import paper_2211_16479_b200 as ms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 7672.0) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 7672.0

n = 1 << 24
base = mi.keys_torch(n, 1, "u31", device="cuda")
for L, rand in ((16, False), (32, True), (100, False), (256, False), (256, True), (1000, False),
                (2176, False), (8704, False), (8704, True), (65536, False), (1 << 20, False)):
    if rand:
        lens = np.random.default_rng(9).integers(1, L + 1, n // max(L // 2, 1) + 16)
        lens = lens[:np.searchsorted(np.cumsum(lens), n) + 1]
        lens[-1] -= lens.sum() - n
    else:
        lens = np.full(n // L, L)
        if lens.sum() < n:
            lens = np.append(lens, n - lens.sum())
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    assert off[-1] == n
    off_dev = torch.from_numpy(off).cuda()
    for pairs, dev in ((False, False), (True, False), (False, True), (True, True)):
        k = base.clone()
        v = torch.arange(n, dtype=torch.int32, device="cuda") if pairs else None
        v0 = v.clone() if pairs else None
        nb = ms.msort_segmented_workspace_bytes(n, off.size - 1, ms.MSORT_INT32,
                                                ms.MSORT_UINT32 if pairs else ms.MSORT_NONE)
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        offs = off_dev if dev else off
        ms.msort_sort_segmented(k, offs, v, ws=ws)
        torch.cuda.synchronize()
        ts, hs = [], []
        for _ in range(a.reps):
            k.copy_(base)
            if pairs:
                v.copy_(v0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            h0 = time.perf_counter()
            ms.msort_sort_segmented(k, offs, v, ws=ws)
            hs.append((time.perf_counter() - h0) * 1e3)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        med = statistics.median(ts)
        ok = True
        for i in np.linspace(0, off.size - 2, 64).astype(int):  # sampled segments sorted
            s = k[off[i]:off[i + 1]]
            ok &= bool((s[1:] >= s[:-1]).all()) if s.numel() > 1 else True
        rec = 4 + (4 if pairs else 0)
        print(json.dumps({"seg_len": ("uniform 1.." if rand else "") + str(L), "nseg": int(off.size - 1),
                          "n": n, "pairs": pairs,
                          "offsets": "device" if dev else "host", "ms": round(med, 4),
                          "host_enqueue_ms": round(statistics.median(hs), 4),
                          "gkeys_s": round(n / med / 1e6, 2),
                          "hbm_floor_frac": round(2 * n * rec / (med / 1e3) / 1e9 / peak, 3),
                          "sorted": ok}), flush=True)
