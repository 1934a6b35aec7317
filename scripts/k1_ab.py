"""A/B of the tile sort (K1) alone: the product kernel (per-thread merge-exchange
network on 68 keys + merge-path rounds in shared memory, T = 8704) vs the
warp-shuffle variant (north_star (1): each warp sorts 32 x 64 keys with the
warp-shuffle bitonic network, then the same block rounds, T = 8192), on 2^28
int32 keys (msort_debug_tile_sort).

    python scripts/k1_ab.py [--log2n 28] [--reps 20]
Prints per variant: median ms, ns per key, and whether every tile came out
sorted with its multiset sum unchanged.
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
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
n = 1 << a.log2n
kin = mi.keys_torch(n, 4, "u31", device="cuda")
kout = torch.empty_like(kin)
st = torch.cuda.current_stream().cuda_stream
for variant in (0, 1):
    T = 0
    for _ in range(3):
        T = ms.lib.msort_debug_tile_sort(ctypes.c_void_p(kin.data_ptr()),
                                         ctypes.c_void_p(kout.data_ptr()), n, variant,
                                         ctypes.c_void_p(st))
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ms.lib.msort_debug_tile_sort(ctypes.c_void_p(kin.data_ptr()),
                                     ctypes.c_void_p(kout.data_ptr()), n, variant,
                                     ctypes.c_void_p(st))
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    full = n // T * T
    v = kout[:full].view(-1, T)
    ok = bool((v[:, 1:] >= v[:, :-1]).all()) and torch.equal(
        v.to(torch.int64).sum(1), kin[:full].view(-1, T).to(torch.int64).sum(1))
    med = statistics.median(ts)
    print(json.dumps({"variant": ["product 128x68 (network + merge rounds)",
                                  "warp-shuffle bitonic 128x64"][variant], "tile": T,
                      "ms": round(med, 4), "ns_per_key": round(med * 1e6 / n, 4),
                      "tiles_sorted": ok}), flush=True)
