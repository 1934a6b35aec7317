"""Median ms of 200 out-of-place int32 sorts at 2^18..2^24 keys (small/mid-size latency A/B)."""
import sys, statistics, json
sys.path.insert(0, '/root/repo')
import torch, msort_inputs as mi, paper_2211_16479_b200 as ms
for lg in (18, 20, 22, 24):
    n = 1 << lg
    kin = mi.keys_torch(n, 1, "u31", device="cuda"); kout = torch.empty_like(kin)
    ws = ms.workspace(n, kin.dtype, False, device="cuda")
    for _ in range(10): ms.msort_sort_out(kin, kout, ws=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(200):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ms.msort_sort_out(kin, kout, ws=ws); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(lg, round(statistics.median(ts), 4))
