"""Quick A/B timing of one library build on C2-shaped inputs (2^24 int32;
random / sorted / reversed) and a few other sizes; sortedness checked against
torch.sort (tuning aid only -- the parity tests compare with the oracle).

    MSORT_LIB=... python scripts/c2_time.py [--log2n 24 20 26]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import msort_inputs as mi  # noqa: E402
import paper_2211_16479_b200 as ms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, nargs="+", default=[24])
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
tag = os.path.basename(os.environ.get("MSORT_LIB", "default"))
for lg in a.log2n:
    n = 1 << lg
    base = mi.keys_torch(n, 1, "u31", device="cuda")
    ref = torch.sort(base).values
    for order in ("random", "sorted", "reversed"):
        kin = base if order == "random" else (ref.clone() if order == "sorted" else ref.flip(0).contiguous())
        kout = torch.empty_like(kin)
        ws = ms.workspace(n, kin.dtype, False, device="cuda")
        for _ in range(3):
            ms.msort_sort_out(kin, kout, ws=ws)
        ok = bool(torch.equal(kout, ref))
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ms.msort_sort_out(kin, kout, ws=ws)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(f"{tag:24s} 2^{lg} {order:8s} med {ts[len(ts) // 2]:8.1f} us  min {ts[0]:8.1f}  ok {ok}")
