"""One call per batched-sort workload, for ncu (scripts/ncu_seg.sh): 2^24 int32
keys as 2^20 x 16 (warp network, device offsets), 7711 x 2176 (CTA tile sort),
256 x 65536 (K1 per tile + the fused segment merge SegFused)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import msort_inputs as mi  # noqa: E402
import paper_2211_16479_b200 as ms  # noqa: E402

n = 1 << 24
base = mi.keys_torch(n, 1, "u31", device="cuda")
for L in (16, 2176, 65536):
    lens = np.full(n // L, L)
    if lens.sum() < n:
        lens = np.append(lens, n - lens.sum())
    off = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)).cuda()
    k = base.clone()
    ms.msort_sort_segmented(k, off)
    torch.cuda.synchronize()
    s = k[: min(L, n)]
    assert bool((s[1:] >= s[:-1]).all())
print("ok")
