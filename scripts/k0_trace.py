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
buf = (ctypes.c_ulonglong * (16 * 32))()
ms.lib.msort_debug_k0_trace(buf)
t = [[buf[c * 32 + s] for s in range(32)] for c in range(16)]
t0 = min(x for row in t for x in row if x > 10**12)  # timestamps (slot 21: a count)
names = {0: "start", 1: "bitonic", 2: "phase1", 3: "cl_sync0", 30: "end", 31: "end_sync"}
if os.environ.get("MSORT_K0", "1") == "1":  # multiway phase 2
    names.update({7: "samples", 8: "ranked", 4: "bounds_sync", 9: "states", 10: "copied",
                  5: "sentinels", 11: "round0", 12: "round1", 13: "round2", 6: "merged",
                  20: "layout", 22: "w0_layout_done", 23: "w1_at_bar"})
else:
    for l in range(4):
        names[4 + 3 * l], names[5 + 3 * l], names[6 + 3 * l] = f"l{l}_search", f"l{l}_copy", f"l{l}_done"
for c in range(16):
    if any(t[c]):
        print(json.dumps({names.get(s, str(s)): (round((t[c][s] - t0) / 1e3, 2) if t[c][s] > t0 else t[c][s])
                          for s in range(32) if t[c][s]}))
