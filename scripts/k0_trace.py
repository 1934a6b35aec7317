"""K0 phase timeline (tuning build -DMSORT_K0_TRACE): globaltimer per CTA.
    MSORT_LIB=.../libmsort_k0trace.so python scripts/k0_trace.py [--log2n 16]"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import msort_inputs as mi  # noqa: E402
import paper_2211_16479_b200 as ms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=16)
a = ap.parse_args()
n = 1 << a.log2n
kin = mi.keys_torch(n, 0, "u31", device="cuda")
kout = torch.empty_like(kin)
for _ in range(5):
    ms.msort_sort_out(kin, kout)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 128)()
ms.lib.msort_debug_k0_trace(buf)
t = [[buf[c * 16 + s] for s in range(16)] for c in range(8)]
t0 = min(x for row in t for x in row if x)
names = ["start", "bitonic", "phase1", "cl_sync0", "l0_search", "l0_merge", "l0_done", "l1_search",
         "l1_merge", "l1_done", "l2_search", "l2_merge", "l2_done", "-", "end", "end_sync"]
for c in range(8):
    print(json.dumps({names[s]: round((t[c][s] - t0) / 1e3, 2) for s in range(16) if t[c][s]}))
