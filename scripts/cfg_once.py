"""Run one BASELINE config through msort_sort_out R times (for ncu captures).
    python scripts/cfg_once.py C3 [--reps 3]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import msort_inputs as mi  # noqa: E402
import paper_2211_16479_b200 as ms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
k, v = mi.config_input(a.config)
kin = torch.from_numpy(k).cuda()
vin = torch.from_numpy(v.view("int32")).cuda().view(torch.uint32) if v is not None else None
if k.dtype.name == "uint32":
    kin = torch.from_numpy(k.view("int32")).cuda().view(torch.uint32)
kout = torch.empty_like(kin)
vout = torch.empty_like(vin) if vin is not None else None
for _ in range(a.reps):
    ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout)
torch.cuda.synchronize()
print("ok", a.config, k.size)
