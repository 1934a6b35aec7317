"""Per-call host cost and back-to-back device time of small sorts (2^12, 2^16, 2^20 int32).

    python scripts/call_latency.py
"""
import sys, time, statistics, json
sys.path.insert(0, '/root/repo')
import torch, msort_inputs as mi, paper_2211_16479_b200 as ms
for lg in (12, 16, 20):
    n = 1 << lg
    kin = mi.keys_torch(n, 0, "u31", device="cuda"); kout = torch.empty_like(kin)
    ws = ms.workspace(n, kin.dtype, False, device="cuda")
    for _ in range(20): ms.msort_sort_out(kin, kout, ws=ws)
    torch.cuda.synchronize()
    # host cost per call
    t0 = time.perf_counter()
    for _ in range(200): ms.msort_sort_out(kin, kout, ws=ws)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    # device time per call, back to back (graph of 20 calls)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200): ms.msort_sort_out(kin, kout, ws=ws)
    e1.record(); e1.synchronize()
    print(json.dumps({"n": n, "host_us_per_call": round((t1 - t0) / 200 * 1e6, 2),
                      "back_to_back_us_per_call": round(e0.elapsed_time(e1) / 200 * 1e3, 2)}))
