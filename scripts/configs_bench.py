"""Time every BASELINE.json config on one GPU (out of place, workspace preallocated),
following SURVEY.md §8(d)'s GPU timing protocol.

    python scripts/configs_bench.py [--reps 20] [--reps-small 100]

C1 2^16 int32 u31 | C2 2^24 int32 (random / sorted / reversed) | C3 2^26 int64 mod 1000 + uint32
index payload | C4 2^27 uint32 + uint32 index payload | C5 2^28 int32 (one shard).
Per repetition: an untimed L2 flush (a write of 2x the L2 size), then CUDA events around the
msort call.  C1/C2 are also timed without the flush (their data fits in L2).  One JSON line per
config: median and min ms, G keys/s, the tile T and pass count P, the BJ roofline fraction
f = t_roof / t_meas with t_roof = every executed pass's 2 n (wk + wv) bytes at the measured HBM
copy bandwidth, the floor fraction (one read + one write), the first call's time including the
workspace allocation, and the outputs checked against torch.sort (keys) / the stable index order.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import msort_inputs as mi  # noqa: E402
import paper_2211_16479_b200 as ms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--reps-small", type=int, default=100)
a = ap.parse_args()

peaks = os.path.join(ROOT, "MEASURED_PEAKS.json")
BW = json.load(open(peaks)).get("hbm_gbs", 6547.5) if os.path.exists(peaks) else 6547.5
L2 = torch.cuda.get_device_properties(0).L2_cache_size
flush_buf = torch.empty(2 * L2 // 4, dtype=torch.int32, device="cuda")


def flush():
    flush_buf.fill_(1)


CFG = [("C1", 16, 0, "u31", False, None), ("C2", 24, 1, "u31", False, None),
       ("C2s", 24, 1, "u31", False, "sorted"), ("C2r", 24, 1, "u31", False, "reversed"),
       ("C3", 26, 2, ("mod", 1000), True, None), ("C4", 27, 3, "u32", True, None),
       ("C5", 28, 4, "u31", False, None)]
res = {}
for name, lg, seed, dist, pairs, variant in CFG:
    n = 1 << lg
    kin = mi.keys_torch(n, seed, dist, device="cuda")
    if variant:
        kin = torch.sort(kin.to(torch.int64))[0].to(kin.dtype)
        if variant == "reversed":
            kin = kin.flip(0).contiguous()
    kout = torch.empty_like(kin)
    vin = torch.arange(n, dtype=torch.int32, device="cuda") if pairs else None
    vout = torch.empty_like(vin) if pairs else None
    # first call, workspace allocation included
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ws = ms.workspace(n, kin.dtype, pairs, device="cuda")
    ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
    torch.cuda.synchronize()
    first_ms = (time.perf_counter() - t0) * 1e3
    for _ in range(3):
        ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
    torch.cuda.synchronize()
    reps = a.reps_small if lg <= 24 else a.reps

    def timed(do_flush):
        ts = []
        for _ in range(reps):
            if do_flush:
                flush()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts), min(ts)

    med, mn = timed(True)
    un = timed(False) if lg <= 24 else None
    # verification: keys equal torch's stable sort, payload its index order
    def as_i64(t):
        if t.dtype == torch.int64:
            return t
        if t.dtype == torch.int32:
            return t.to(torch.int64)
        return t.view(torch.int32).to(torch.int64) & 0xFFFFFFFF  # uint32

    ref = torch.sort(as_i64(kin), stable=True)
    ok = bool(torch.equal(as_i64(kout), ref[0]))
    if pairs:
        ok &= bool(torch.equal(vout.to(torch.int64), ref[1]))
    del ref
    kd = ms.MSORT_INT64 if kin.dtype == torch.int64 else ms.MSORT_INT32
    T = ms.tile_size(kd, ms.MSORT_UINT32 if pairs else ms.MSORT_NONE)
    P = 1 + (((n + T - 1) // T) - 1).bit_length()  # K1 pass + merge levels
    rec = kin.element_size() + (4 if pairs else 0)
    t_roof = P * 2 * n * rec / (BW * 1e9) * 1e3
    t_floor = 2 * n * rec / (BW * 1e9) * 1e3
    line = {"config": name, "n": n, "pairs": pairs, "ms_median": round(med, 4),
            "ms_min": round(mn, 4), "gkeys_s": round(n / med / 1e6, 3), "tile": T, "passes": P,
            "roofline_frac": round(t_roof / med, 3), "floor_frac": round(t_floor / med, 4),
            "first_call_ms_incl_alloc": round(first_ms, 3), "l2_flushed": True,
            "verified": ok, "reps": reps, "hbm_gbs": BW, "l2_bytes": L2}
    if un:
        line["ms_median_unflushed"], line["ms_min_unflushed"] = round(un[0], 4), round(un[1], 4)
    res[name] = med
    print(json.dumps(line), flush=True)
    del kin, kout, vin, vout, ws
    torch.cuda.empty_cache()
print(json.dumps({"P142_check": "merge sort unaffected by the initial order (P:142)",
                  "t_C2s_over_t_C2": round(res["C2s"] / res["C2"], 3),
                  "t_C2r_over_t_C2": round(res["C2r"] / res["C2"], 3)}), flush=True)
