"""Distributed sort in the one-GPU emulation (p virtual ranks, same kernels):
time per call for both exchange modes (include/msort.h msort_debug_set_exchange)
and for the paper's rank-tree gather to rank 0 (msort_sort_distributed_tree,
mode "tree": the root ends with all p * n keys).

    python scripts/dist_emul_bench.py [--log2n 26] [--ps 2,4,8] [--reps 5]
All p ranks run on one GPU in sequence, so the time is p x (one rank's work)
plus the emulated collectives; the exchange in mode 0 is a D2D copy, in mode 1
the first merge round reads the other "ranks'" buffers directly.
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
ap.add_argument("--log2n", type=int, default=26)
ap.add_argument("--ps", default="2,4,8")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
n = 1 << a.log2n
for p in [int(x) for x in a.ps.split(",")]:
    src = [mi.keys_torch(n, 4 + r, "u31", device="cuda") for r in range(p)]
    for mode in (0, 1):
        ms.set_exchange_mode(mode)
        ts = []
        for rep in range(a.reps + 2):
            kd = [s.clone() for s in src]
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            if rep == 2:
                ms.profile_reset()
                ms.profile_enable(True)
            e0.record()
            ms.msort_sort_distributed_emulated(kd)
            e1.record()
            e1.synchronize()
            if rep == 2:
                ms.profile_enable(False)
                phases = {k: round(v[1], 3) for k, v in ms.profile_read().items() if v[0]}
            if rep >= 2:
                ts.append(e0.elapsed_time(e1))
        ok = all(bool((k[1:] >= k[:-1]).all()) for k in kd)
        med = statistics.median(ts)
        print(json.dumps({"p": p, "n_per_rank": n, "mode": ["alltoall", "pull"][mode],
                          "ms_all_ranks": round(med, 3), "ms_per_rank": round(med / p, 3),
                          "phases_ms_all_ranks": phases, "sorted": ok}), flush=True)
        del kd
    ms.set_exchange_mode(0)
    # the paper's rank-tree gather (all data ends on the root)
    ts = []
    for rep in range(a.reps + 2):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        rk, _ = ms.msort_sort_distributed_tree_emulated(src)
        e1.record()
        e1.synchronize()
        if rep >= 2:
            ts.append(e0.elapsed_time(e1))
    ok = bool((rk[1:] >= rk[:-1]).all())
    med = statistics.median(ts)
    print(json.dumps({"p": p, "n_per_rank": n, "mode": "tree", "ms_all_ranks": round(med, 3),
                      "ms_per_rank": round(med / p, 3), "sorted": ok}), flush=True)
    del rk
    del src
    torch.cuda.empty_cache()
