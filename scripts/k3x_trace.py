"""Wait-time breakdown of one K3X pass (tuning build with -DMSORT_K3X_TRACE).

    python paper_2211_16479_b200/build.py -D MSORT_K3X_TRACE=1 --out /tmp/x.so
    MSORT_LIB=/tmp/x.so MSORT_QUAD=4 python scripts/k3x_trace.py
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import msort_inputs as mi  # noqa: E402
import paper_2211_16479_b200 as ms  # noqa: E402

n = 1 << 28
kin = mi.keys_torch(n, 4, "u31", device="cuda")
kout = torch.empty_like(kin)
ws = ms.workspace(n, kin.dtype, False, device="cuda")
buf = (ctypes.c_ulonglong * (1024 * 8))()
for _ in range(2):
    ms.msort_sort_out(kin, kout, ws=ws)
torch.cuda.synchronize()
ms.lib.msort_debug_k3x_trace(buf, 1024 * 8, 1)
ms.msort_sort_out(kin, kout, ws=ws)
torch.cuda.synchronize()
ms.lib.msort_debug_k3x_trace(buf, 1024 * 8, 0)
t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8).astype(np.float64)
t = t[t[:, 6] > 0]
names = ["mergers wait full", "producer wait searcher", "producer wait store", "searcher wait ring",
         "store wait mergers", "span (all passes)", "tiles"]
print("CTAs", len(t))
for i, nm in enumerate(names):
    col = t[:, i]
    sc = 1 if i == 6 else 1e6
    print(f"{nm:24s} mean {col.mean()/sc:10.3f} max {col.max()/sc:10.3f}  ({'ms' if i < 6 else 'n'})")
