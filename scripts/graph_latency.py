"""Small-sort latency: direct calls vs one CUDA graph replay of the same call.

    python scripts/graph_latency.py [--sizes 13,16,18,20] [--reps 200]
The sort is asynchronous and allocation-free with a preallocated workspace,
so torch.cuda.graph can capture it (memset + K1 + fused K3 launches).
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
ap.add_argument("--sizes", default="13,16,18,20")
ap.add_argument("--reps", type=int, default=200)
a = ap.parse_args()


def timeit(fn, reps):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


for lg in [int(x) for x in a.sizes.split(",")]:
    n = 1 << lg
    kin = mi.keys_torch(n, 0, "u31", device="cuda")
    kout = torch.empty_like(kin)
    ws = ms.workspace(n, kin.dtype, False, device="cuda")
    s = torch.cuda.Stream()
    direct = timeit(lambda: ms.msort_sort_out(kin, kout, ws=ws), a.reps)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        ms.msort_sort_out(kin, kout, ws=ws, stream=s)  # warm (lazy init outside capture)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            ms.msort_sort_out(kin, kout, ws=ws, stream=s)
    kout.zero_()
    graph = timeit(g.replay, a.reps)
    ok = bool((kout[1:] >= kout[:-1]).all()) and int(kout.sum(dtype=torch.int64)) == int(
        kin.sum(dtype=torch.int64))
    print(json.dumps({"log2n": lg, "direct_us": round(direct * 1e3, 1),
                      "graph_us": round(graph * 1e3, 1), "sorted": ok}), flush=True)
