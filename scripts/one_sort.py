"""Run one input through msort_sort_out R times (for ncu captures).

    python scripts/one_sort.py --log2n 24 --order random --reps 4
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
ap.add_argument("--log2n", type=int, default=24)
ap.add_argument("--order", default="random", choices=["random", "sorted", "reversed"])
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
n = 1 << a.log2n
kin = mi.keys_torch(n, a.seed, "u31", device="cuda")
if a.order != "random":
    kin = torch.sort(kin, descending=a.order == "reversed").values
kout = torch.empty_like(kin)
ws = ms.workspace(n, kin.dtype, False, device="cuda")
for _ in range(a.reps):
    ms.msort_sort_out(kin, kout, ws=ws)
torch.cuda.synchronize()
print("ok", a.log2n, a.order)
