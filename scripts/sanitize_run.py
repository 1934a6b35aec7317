"""Small workloads for compute-sanitizer (memcheck): every kernel path once.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py
keys (int32, int64) and pairs sorts with ragged tails, the 4-way K3Q path,
out-of-place misaligned views, and the emulated distributed sort in both
exchange modes.  Exits non-zero on a wrong result.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import msort_inputs as mi  # noqa: E402
import paper_2211_16479_b200 as ms  # noqa: E402


def check_sorted(t):
    assert bool((t[1:] >= t[:-1]).all())


for dist, n in (("i32", 300001), ("i64", 200003), ("u31", 1 << 18)):
    k = mi.keys_torch(n, 3, dist, device="cuda")
    ms.msort_sort(k)
    check_sorted(k)
k = mi.keys_torch(250007, 4, "u31", device="cuda")
v = torch.arange(k.numel(), dtype=torch.int32, device="cuda")
ms.msort_sort_pairs(k, v)
check_sorted(k)
ms.set_quad_mode(5)
k = mi.keys_torch(300001, 5, "u31", device="cuda")
ms.msort_sort(k)
check_sorted(k)
ms.set_quad_mode(0)
base = mi.keys_torch(200001, 6, "u31", device="cuda")
kin = base[1:]
kout = torch.empty(200003, dtype=torch.int32, device="cuda")[3:3 + kin.numel()]
ms.msort_sort_out(kin.contiguous() if False else kin, kout)
check_sorted(kout)
for mode in (0, 1):
    ms.set_exchange_mode(mode)
    kd = [mi.keys_torch(60000 + 1000 * r, 10 + r, "u31", device="cuda") for r in range(3)]
    vd = [torch.arange(x.numel(), dtype=torch.int32, device="cuda") for x in kd]
    ms.msort_sort_distributed_emulated(kd, vd)
    for x in kd:
        check_sorted(x)
ms.set_exchange_mode(0)
torch.cuda.synchronize()
print("sanitize workload ok")

# batched sorts (every length bin, host and device offsets), K6 mode, rank tree
import numpy as np  # noqa: E402

lens = [0, 1, 7, 32, 33, 100, 256, 1000, 2176, 5000, 8704, 20000, 3]
off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
for dev_off in (False, True):
    k = mi.keys_torch(int(off[-1]), 6, "u31", device="cuda")
    v = torch.arange(k.numel(), dtype=torch.int32, device="cuda")
    ms.msort_sort_segmented(k, torch.from_numpy(off).cuda() if dev_off else off, v)
    for i in range(len(lens)):
        check_sorted(k[off[i]:off[i + 1]]) if lens[i] > 1 else None
ms.set_quad_mode(5)
k = mi.keys_torch(8704 * 40 + 5, 7, "u31", device="cuda")
ms.msort_sort(k)
check_sorted(k)
ms.set_quad_mode(0)
rk, _ = ms.msort_sort_distributed_tree_emulated(
    [mi.keys_torch(50000 + r, 8 + r, "u31", device="cuda") for r in range(3)])
check_sorted(rk)
torch.cuda.synchronize()
print("sanitize workload ok")
