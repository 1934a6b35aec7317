"""Per-CTA timeline of the last K3 launch (tuning builds with -DMSORT_K3_TRACE).

    python paper_2211_16479_b200/build.py -D MSORT_K3_TRACE=1 --out /tmp/trace.so
    MSORT_LIB=/tmp/trace.so python scripts/k3_trace.py [--log2n 28]
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
ap.add_argument("--log2n", type=int, default=28)
a = ap.parse_args()
n = 1 << a.log2n
kin = mi.keys_torch(n, 4, "u31", device="cuda")
kout = torch.empty_like(kin)
ws = ms.workspace(n, kin.dtype, False, device="cuda")
for _ in range(3):
    ms.msort_sort_out(kin, kout, ws=ws)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4096 * 8))()
ms.lib.msort_debug_k3_trace(buf, 4096 * 8)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).astype(np.int64)
t = t[t[:, 5] > 0]
start = t[:, 0] - t[:, 0].min()
names = ["start(us)", "chunk0 coranks", "after grab", "first full", "end", "tiles",
         "consumer wait", "producer wait"]
print("CTAs", len(t))
for i, nm in enumerate(names):
    col = start if i == 0 else t[:, i]
    sc = 1 if i == 5 else 1e3
    print(f"{nm:15s} min {col.min()/sc:10.2f} med {np.median(col)/sc:10.2f} max {col.max()/sc:10.2f}")
end_abs = start + t[:, 4]
print(f"kernel span (first start -> last end) {end_abs.max()/1e3:.1f} us")
