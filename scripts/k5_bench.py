"""D4 merge A/B: K5 (one pass) vs K3 rounds, through msort_merge_runs.

    python scripts/k5_bench.py [--log2n 28] [--ps 3,4,8,16] [--reps 10]
    MSORT_K5=0 python scripts/k5_bench.py ...      (K3 rounds, for the A/B)

The C5 shape of D4 at p ranks: n = 2^28 int32 keys on one rank, in p runs of
n/p keys each (sorted uniform [0, 2^31) segments).  Prints per p: median ms of
the call (CUDA events; inputs > L2), the per-class device times (partition =
sampling + sample merge + tile states, kway = the K5 merge or the K3 rounds),
achieved GB/s of the merge kernel on 2 n wk algorithmic bytes, and whether the
output is sorted with the input's sum.
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
ap.add_argument("--log2n", type=int, default=28)
ap.add_argument("--ps", default="3,4,8,16")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
n = 1 << a.log2n
for p in [int(x) for x in a.ps.split(",")]:
    per = n // p
    off = [j * per for j in range(p)] + [n]
    kin = mi.keys_torch(n, 4, "u31", device="cuda")
    for j in range(p):  # sorted runs
        kin[off[j]:off[j + 1]] = torch.sort(kin[off[j]:off[j + 1]])[0]
    kout = torch.empty_like(kin)
    nb = ms.ctypes.c_size_t()
    ms.lib.msort_merge_runs_workspace_bytes(n, p, ms.MSORT_INT32, ms.MSORT_NONE, ms.ctypes.byref(nb))
    ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ms.msort_merge_runs(kin, off, kout, ws=ws)
    torch.cuda.synchronize()
    ts = []
    ms.profile_reset()
    ms.profile_enable(True)
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ms.msort_merge_runs(kin, off, kout, ws=ws)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms.profile_enable(False)
    prof = ms.profile_read()
    ok = bool((kout[1:] >= kout[:-1]).all()) and int(kout.sum(dtype=torch.int64)) == int(
        kin.sum(dtype=torch.int64))
    kw = prof["kway_merge"]
    part = prof["partition"]
    med = statistics.median(ts)
    print(json.dumps({
        "p": p, "n": n, "k5": os.environ.get("MSORT_K5", "1") != "0", "ms": round(med, 4),
        "min_ms": round(min(ts), 4),
        "merge_ms": round(kw[1] / a.reps, 4), "merge_launches": kw[0] / a.reps,
        "partition_ms": round(part[1] / a.reps, 4), "partition_launches": part[0] / a.reps,
        "merge_gbs_2nwk": round(2 * n * 4 / (kw[1] / kw[0] * kw[0] / a.reps / 1e3) / 1e9, 1)
        if kw[0] else None,
        "call_gbs_2nwk": round(2 * n * 4 / (med / 1e3) / 1e9, 1), "ok": ok}), flush=True)
    del kin, kout, ws
    torch.cuda.empty_cache()
