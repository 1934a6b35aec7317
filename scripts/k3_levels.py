"""Per-level timeline of the fused K3 launch (tuning builds with -DMSORT_K3_TRACE).

    python paper_2211_16479_b200/build.py -D MSORT_K3_TRACE=1 --out build_trace/libmsort_trace.so
    MSORT_LIB=build_trace/libmsort_trace.so python scripts/k3_levels.py --log2n 24 [--order sorted]

For every merge level: when its first chunk was grabbed, when its first / last
chunk had its inputs ready, how long the co-rank searches took, and when its
first / last tile was published (us from the first grab of the launch).
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import msort_inputs as mi  # noqa: E402
import paper_2211_16479_b200 as ms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=24)
ap.add_argument("--order", default="random", choices=["random", "sorted", "reversed"])
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
n = 1 << a.log2n
kin = mi.keys_torch(n, a.seed, "u31", device="cuda")
if a.order == "sorted":
    kin = torch.sort(kin).values
elif a.order == "reversed":
    kin = torch.sort(kin, descending=True).values
kout = torch.empty_like(kin)
ws = ms.workspace(n, kin.dtype, False, device="cuda")
for _ in range(3):
    ms.msort_sort_out(kin, kout, ws=ws)
torch.cuda.synchronize()
ms.lib.msort_debug_k3_trace_clear()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ms.msort_sort_out(kin, kout, ws=ws)
e1.record()
torch.cuda.synchronize()
print(f"n=2^{a.log2n} {a.order}: sort {e0.elapsed_time(e1) * 1e3:.1f} us (traced build)")
NT, NC = 1 << 20, 1 << 18
tiles = (ctypes.c_ulonglong * NT)()
chunks = (ctypes.c_ulonglong * (NC * 4))()
assert ms.lib.msort_debug_k3_trace2(tiles, NT, chunks, NC) == 0
t = np.frombuffer(tiles, dtype=np.uint64).astype(np.int64)
c = np.frombuffer(chunks, dtype=np.uint64).astype(np.int64).reshape(NC, 4)
T = ms.tile_size(ms.MSORT_INT32, ms.MSORT_NONE) if hasattr(ms, "MSORT_NONE") else 8704
Tm = 8704
ntiles = (n + Tm - 1) // Tm
P = int(np.ceil(np.log2(n / T)))
CH = max(1, min(8, ntiles // (2 * 148 * 2)))  # chunk_tiles (2 CTAs/SM)
cpp = (ntiles + CH - 1) // CH
nch = P * cpp
c = c[:nch]
t0 = c[c[:, 0] > 0, 0].min()
print(f"chunk {CH} tiles; tiles/level {ntiles}, levels {P}, chunks/level {cpp}, CTAs {len(np.unique(c[:, 3]))}")
print(f"{'lvl':>3} {'grab0':>8} {'rdy0':>8} {'rdyN':>8} {'srch med':>8} {'wait med':>8} "
      f"{'wait max':>8} {'done0':>8} {'doneN':>8} {'span':>7}")
for p in range(P):
    cc = c[p * cpp:(p + 1) * cpp]
    tt = t[p * ntiles:(p + 1) * ntiles]
    ok = cc[:, 0] > 0
    if not ok.any():
        continue
    cc = cc[ok]
    g, r, s = (cc[:, 0] - t0) / 1e3, (cc[:, 1] - t0) / 1e3, (cc[:, 2] - t0) / 1e3
    d = (tt[tt > 0] - t0) / 1e3
    print(f"{p:3d} {g.min():8.1f} {r.min():8.1f} {r.max():8.1f} {np.median(s - r):8.2f} "
          f"{np.median(r - g):8.2f} {(r - g).max():8.2f} {d.min():8.1f} {d.max():8.1f} "
          f"{d.max() - d.min():7.1f}")
