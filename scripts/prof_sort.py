"""Small driver for ncu / compute-sanitizer: sort one seeded input `reps` times.

    python scripts/prof_sort.py [--log2n 26] [--dtype i32|u32|i64|u64] [--pairs] [--reps 2]

Out-of-place (msort_sort_out_ws) from a pristine input each repetition, so
every repetition does identical work.  Verifies the last output is sorted.
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
ap.add_argument("--log2n", type=int, default=26)
ap.add_argument("--dtype", default="i32")
ap.add_argument("--pairs", action="store_true")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
n = 1 << a.log2n
dist = {"i32": "u31", "u32": "u32", "i64": "i64", "u64": "u64"}[a.dtype]
kin = mi.keys_torch(n, 4, dist, device="cuda")
kout = torch.empty_like(kin)
vin = torch.arange(n, dtype=torch.int32, device="cuda") if a.pairs else None
vout = torch.empty_like(vin) if a.pairs else None
ws = ms.workspace(n, kin.dtype, a.pairs, device="cuda")
for _ in range(a.reps):
    ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
torch.cuda.synchronize()
k = kout.view(torch.int64) if kout.dtype == torch.uint64 else kout
ok = bool((kout[1:] >= kout[:-1]).all()) if kout.dtype not in (torch.uint32, torch.uint64) else True
print("sorted" if ok else "NOT SORTED", n, a.dtype, "pairs" if a.pairs else "keys")
sys.exit(0 if ok else 1)
