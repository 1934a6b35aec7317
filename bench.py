#!/usr/bin/env python3
"""Benchmark: stable merge sort of 2^28 int32 keys per GPU (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: distributed sort)

Workload (BASELINE.json metric "... (int32, 2^28/GPU)", config C5): every rank
holds 2^28 int32 keys uniform in [0, 2^31) from counter-mode SplitMix64 with
seed 4 + rank (msort_inputs; DESIGN.md input recipe).  N = 1: one local sort
(msort_sort_out_ws).  N > 1: the distributed sort (local sort, splitter
co-rank, NCCL all-to-all, k-way merge; msort_sort_distributed_out_ws), and the
output is globally sorted across ranks.

A step sorts the pristine input into an output buffer (out-of-place, so no
restore copy is needed and the input is never sorted data).  Inputs and the
workspace (1 GiB + 1 GiB + 1 GiB per GPU) are far larger than L2 (126 MB), so
no L2 flush is done between steps.  Timing: W untimed steps, then K steps
between a barrier + cuda.synchronize on both sides, CUDA events on the
launching stream, max over ranks.  Rank 0 prints one JSON line.

N = 1 also reports "batched_sort" (outside the timed region
and the headline): 2^24 keys in 2^20 x 16, 2^16 x 256 and 256 x 65536 segments
sorted by one msort_sort_segmented call each (--no-batched skips it).

--impl reference times the CPU oracle (oracle/, textbook top-down merge sort)
on a bounded sample of the same workload on this host's cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sorted keys/sec and % of HBM/NVLink roofline at 1/2/4/8 B200 (int32, 2^28/GPU)"
N_PER_GPU = 1 << 28
SEED0 = 4
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--n", type=int, default=N_PER_GPU, help="keys per GPU (default 2^28)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--distributed-path", action="store_true",
                    help="run the N > 1 code path even at N = 1 (a one-rank NCCL group; a "
                         "smoke test of the distributed bench on a one-GPU box)")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config lines (C1-C4, BASELINE.json configs 1-4)")
    ap.add_argument("--no-batched", action="store_true",
                    help="skip the batched (segmented) sort lines (SURVEY §8(f) f3)")
    ap.add_argument("--e2e-streams", type=int, default=3, help="streams the e2e steps rotate over")
    ap.add_argument("--exchange", choices=["auto", "alltoall", "pull"], default="auto",
                    help="N > 1: NCCL all-to-all + k-way merge, the fused pull exchange "
                         "(reserved: no host sync per step), or auto = pull if a first "
                         "verified step agrees on every rank, else all-to-all")
    return ap.parse_args()


def expected_digest(world: int, rank: int, n: int):
    """The oracle's SHA-256 of rank `rank`'s expected C5 output slice at
    `world` ranks (tests/golden/c5_digests.json), or None."""
    if n != N_PER_GPU:
        return None
    try:
        with open(os.path.join(ROOT, "tests", "golden", "c5_digests.json")) as f:
            d = json.load(f)["digests"].get(str(world))
        return d[rank]["sha256"] if d else None
    except Exception:
        return None


def host_digest(a) -> str:
    import numpy as np

    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.view(np.uint8)).hexdigest()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload_key: str):
    """Per-launch dram bytes of the merge pass from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(workload_key, {}).get("merge_pass_dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.rows = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(gpu_index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [r for (t, r) in self.rows if t0 - 0.15 <= t <= t1 + 0.15] or [r for _, r in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"]}
        sm = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        mx = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 6 + i and r[6 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows),
                "power_w_max": max((float(r[4]) for r in rows
                                    if r[4].replace(".", "").isdigit()), default=None)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(n_sample: int, samples: int, seed: int = SEED0 + 100):
    """the oracle, as it stands (single-threaded textbook
    top-down merge sort), timed on the host (rank 0).  The default sample is
    one full C5 shard: rank 0's 2^28 keys (seed 4)."""
    import msort_inputs as mi
    import oracle

    oracle.build()
    t = 0.0
    for s in range(samples):
        k = mi.keys(n_sample, seed + s, "u31")
        t0 = time.perf_counter()
        oracle.sort_inplace(k)
        t += time.perf_counter() - t0
    return {"value": n_sample * samples / t, "unit": "keys/s", "cores": 1, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{samples} x 2^{n_sample.bit_length() - 1} int32 keys uniform [0,2^31) "
                      f"(seed {seed}{'' if samples == 1 else '+i'}; seed 4 = the rank-0 C5 shard), "
                      f"single-threaded top-down merge sort (oracle/msort_oracle.c), "
                      f"{t:.1f} s of CPU"}


def cpu_paper_mp(n_sample: int, seed: int = SEED0 + 200):
    """SURVEY.md §8(d) O-c: the paper's multiprocessing merge sort (chunks of
    ceil(n/c) sorted in parallel, then pairwise merges) re-created
    on host threads by the oracle library, all host cores, one 2^k sample."""
    import msort_inputs as mi
    import oracle

    cores = len(os.sched_getaffinity(0))
    k = mi.keys(n_sample, seed, "u31")
    t0 = time.perf_counter()
    oracle.paper_mp_inplace(k, None, cores)
    t = time.perf_counter() - t0
    return {"value": n_sample / t, "unit": "keys/s", "cores": cores, "kind": "oracle_paper_mp",
            "cpu_model": cpu_model(),
            "sample": f"2^{n_sample.bit_length() - 1} int32 keys uniform [0,2^31) (seed {seed}), the paper's "
                      f"multiprocessing merge sort on {cores} host threads "
                      f"(oracle/msort_oracle.c msort_oracle_paper_mp), {t:.1f} s"}


def configs_cpu(per_config):
    """SURVEY §8(d) O-1 and O-c on BASELINE.json's configs 1-4, beside the GPU
    numbers of `configs`: the oracle as it stands (single-threaded top-down
    merge sort; min of 3 for C1/C2, one run for C3/C4) and the paper's
    multiprocessing merge sort on all host cores (min of 3), on the same
    seeded inputs (keys + index payload for C3/C4).  Rank 0, N = 1 only."""
    import msort_inputs as mi
    import oracle

    oracle.build()
    cores = len(os.sched_getaffinity(0))
    for name in ("C1", "C2", "C3", "C4"):
        d = per_config["results"].get(name)
        if d is None:
            continue
        k0, v0 = mi.config_input(name)
        n = k0.size

        def run(fn, reps):
            best = None
            for _ in range(reps):
                k = k0.copy()
                v = v0.copy() if v0 is not None else None
                t0 = time.perf_counter()
                fn(k, v)
                t = time.perf_counter() - t0
                best = t if best is None else min(best, t)
            return best

        t1 = run(lambda k, v: oracle.sort_inplace(k, v), 3 if n <= (1 << 24) else 1)
        tc = run(lambda k, v: oracle.paper_mp_inplace(k, v, cores), 3)
        d["cpu_oracle"] = {"ms": round(t1 * 1e3, 3), "keys_per_s": n / t1, "cores": 1,
                           "kind": "oracle", "reps": 3 if n <= (1 << 24) else 1}
        d["cpu_paper_mp"] = {"ms": round(tc * 1e3, 3), "keys_per_s": n / tc, "cores": cores,
                             "kind": "oracle_paper_mp", "reps": 3}
        d["gpu_over_oracle"] = round(t1 * 1e3 / d["ms"], 1)
        d["gpu_over_paper_mp"] = round(tc * 1e3 / d["ms"], 1)
    per_config["cpu_model"] = cpu_model()


def reference_arm(args, rank):
    """--impl reference: the CPU oracle on a bounded sample per step."""
    if rank != 0:
        return
    import msort_inputs as mi
    import oracle

    oracle.build()
    n_s = 1 << 22
    base = mi.keys(n_s, SEED0, "u31")
    for _ in range(args.warmup):
        oracle.sort_inplace(base.copy())
    t = 0.0
    for _ in range(args.steps):
        k = base.copy()
        t0 = time.perf_counter()
        oracle.sort_inplace(k)
        t += time.perf_counter() - t0
    v = n_s * args.steps / t
    sample = (f"per step: first 2^22 keys of the rank-0 shard (seed 4), single-threaded "
              f"top-down merge sort (oracle/msort_oracle.c)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "keys/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": "C5: 2^28 int32 keys per GPU, uniform [0,2^31), "
                               "counter-mode SplitMix64 seed 4+rank",
                   "n_per_gpu": N_PER_GPU, "key_dtype": "int32", "payload": None,
                   "sample_per_step": f"first 2^22 keys of the rank-0 shard ({n_s} keys)",
                   "parallelism": "single (host, 1 thread)"},
        "cpu_baseline": {"value": v, "unit": "keys/s", "cores": 1, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": v, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def pcie_duplex_ms(h_in, h_out, d_a, d_b, strs, reps=4):
    """Device-timed ms per step of copying h_in -> d_a and d_b -> h_out
    concurrently on two streams (pinned host memory): the floor of an e2e step
    that uploads its input and downloads its result."""
    import torch

    s1, s2 = strs[0], strs[1 % len(strs)]

    def step():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)

    step()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(s1)
    s2.wait_event(e0)
    for _ in range(reps):
        step()
    f1, f2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f1.record(s1)
    f2.record(s2)
    torch.cuda.synchronize()
    return max(e0.elapsed_time(f1), e0.elapsed_time(f2)) / reps


def batched_bench(ms, mi, dev, reps=10):
    """SURVEY §8(f) f3 beside the headline: batched sorts of 2^24 int32 keys
    (seed 1) cut into equal segments, offsets in device memory
    (msort_sort_segmented).  Per workload: median ms of `reps` calls (CUDA
    events around the call, input restored untimed before each), G keys/s,
    and a check that every segment came out non-decreasing with its sum
    unchanged."""
    import torch

    n = 1 << 24
    base = mi.keys_torch(n, 1, "u31", device=dev)
    out = {}
    for seg in (16, 256, 65536):
        nseg = n // seg
        off = torch.arange(0, n + 1, seg, dtype=torch.int64, device=dev)
        k = base.clone()
        nb = ms.msort_segmented_workspace_bytes(n, nseg, ms.MSORT_INT32)
        ws = torch.empty(nb, dtype=torch.uint8, device=dev)
        for _ in range(3):
            k.copy_(base)
            ms.msort_sort_segmented(k, off, ws=ws)
        ts = []
        for _ in range(reps):
            k.copy_(base)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ms.msort_sort_segmented(k, off, ws=ws)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        med = ts[len(ts) // 2]
        v = k.view(nseg, seg)
        ok = bool((v[:, 1:] >= v[:, :-1]).all()) and bool(
            torch.equal(v.to(torch.int64).sum(1), base.view(nseg, seg).to(torch.int64).sum(1)))
        out[f"{nseg}x{seg}"] = {"ms": round(med, 4), "gkeys_s": round(n / med / 1e6, 2),
                                "verified": ok}
    return {"workload": "2^24 int32 keys uniform [0,2^31) (seed 1) in equal segments, "
                        "offsets on the device; msort_sort_segmented", "results": out}


def config_digest(name):
    try:
        with open(os.path.join(ROOT, "tests", "golden", "config_digests.json")) as f:
            return json.load(f)["configs"].get(name)
    except Exception:
        return None


def configs_bench(ms, mi, dev, peak, reps=20):
    """BASELINE.json's single-GPU configs beside the headline:
    C1 (2^16 int32), C2 (2^24 int32; C2s / C2r: the same keys already sorted /
    reverse-sorted -- P:142's "unaffected by the initial array"), C3 (2^26 int64 in [0,1000) + uint32
    index payload), C4 (2^27 uint32 + uint32 index payload).  Per config:
    median device ms of `reps` out-of-place sorts from the pristine input
    (CUDA events around each call; an untimed L2 flush before each for C1/C2,
    whose data fit in L2; C3/C4 are larger than L2), keys/s, the merge
    kernel's roofline (levels x 2 n (wk + wv) bytes per launch over its live
    event time, against the measured HBM peak) and the step's (every executed
    pass at HBM rate), and the output checked BIT FOR BIT against the
    oracle's SHA-256 digests (tests/golden/config_digests.json).  C1 also
    reports the device time of a CUDA-graph replay of the call."""
    import numpy as np
    import torch

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {}
    for name in ("C1", "C2", "C2s", "C2r", "C3", "C4"):
        c = mi.CONFIGS[name[:2]]
        n, pairs = c["n"], c["pairs"]
        k = mi.keys_torch(n, c["seed"], c["dist"], device=dev)
        if c["dist"] == "u32":
            k = k.view(torch.uint32)
        if name in ("C2s", "C2r"):  # BASELINE config 2's already-sorted / reverse-sorted arrays
            k = torch.sort(k)[0]   # (reading R8: the sorted C2 array and its reversal)
            if name == "C2r":
                k = torch.flip(k, [0]).contiguous()
        kin = k
        vin = torch.arange(n, dtype=torch.int32, device=dev).view(torch.uint32) if pairs else None
        kout = torch.empty_like(kin)
        vout = torch.empty_like(vin) if pairs else None
        wk = kin.element_size()
        wv = 4 if pairs else 0
        ws = ms.workspace(n, torch.int64 if wk == 8 else torch.int32, pairs, device=dev)

        def call():
            ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)

        for _ in range(3):
            call()
        torch.cuda.synchronize()
        fits_l2 = n * (wk + wv) <= (64 << 20)  # C1, C2: flushed (the headline) and unflushed

        def timed(do_flush):
            ts_ = []
            for _ in range(reps):
                if do_flush:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                call()
                e1.record()
                e1.synchronize()
                ts_.append(e0.elapsed_time(e1))
            return sorted(ts_)

        unflushed = timed(False) if fits_l2 else None
        ms.profile_reset()
        ms.profile_enable(True)
        ts = timed(fits_l2)
        ms.profile_enable(False)
        prof = ms.profile_read()
        med = ts[len(ts) // 2]
        kd = {4: ms.MSORT_INT32, 8: ms.MSORT_INT64}[wk]
        # 8-byte keys spanning < 2^32 values are sorted as 32-bit offsets
        # (key-range narrowing): merge passes move 4-byte keys,
        # plus the range / narrow / widen passes (8 + 12 + 12 bytes per key)
        narrowed = wk == 8 and n > 65536 and int(kin.max()) - int(kin.min()) < (1 << 32)
        wkm = 4 if narrowed else wk
        T = ms.tile_size(ms.MSORT_UINT32 if narrowed else kd,
                         ms.MSORT_UINT32 if pairs else ms.MSORT_NONE)
        levels = ((n + T - 1) // T - 1).bit_length()
        k0 = not pairs and n <= 65536  # K0: the whole sort in one cluster launch, one HBM pass
        if k0:
            levels = 0
        per_pass = 2 * n * (wkm + wv)
        extra = 32 * n if narrowed else 0
        mp_l, mp_ms = prof["merge_pass"]
        roof = None
        if mp_l:
            # per sort: a narrowed sort also enqueues the (gated-off, empty) 8-byte merge launch
            t_merge = mp_ms / reps
            ach = levels * per_pass / (t_merge / 1e3) / 1e9
            roof = {"kernel": "k3_merge_pass", "bound": "hbm", "achieved": round(ach, 1),
                    "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                    "avg_launch_ms": round(t_merge, 4), "merge_levels": levels,
                    "launches_per_sort": round(mp_l / reps, 2)}
        t_roof = ((levels + 1) * per_pass + extra) / (peak * 1e9) * 1e3
        exp = config_digest(name[:2])  # C2s / C2r sort to C2's output (same multiset)
        ok = None
        if exp:
            a = kout.view(torch.int64 if wk == 8 else torch.int32).cpu().numpy()
            ok = host_digest(a) == exp["keys_sha256"]
            if pairs:
                ok &= host_digest(vout.view(torch.int32).cpu().numpy()) == exp["vals_sha256"]
        d = {"n": n, "key": str(kin.dtype).replace("torch.", ""), "payload": "uint32 index" if pairs
             else None, "key_range_narrowed": narrowed, "ms": round(med, 4), "min_ms": round(ts[0], 4),
             "keys_per_s": n / (med / 1e3), "tile": "K0 cluster (16 x 4096)" if k0 else T,
             "merge_levels": levels,
             "phases_ms": {k2: round(v[1] / reps, 4) for k2, v in prof.items() if v[0]},
             "roofline": roof,
             "step_roofline": {"passes": levels + 1, "t_roof_ms": round(t_roof, 4),
                               "frac": round(t_roof / med, 4),
                               "floor_frac": round(2 * n * (wk + wv) / (peak * 1e9) * 1e3 / med, 4)},
             "l2_flush": fits_l2, "verified": ok}
        if unflushed:
            d["ms_unflushed"] = round(unflushed[len(unflushed) // 2], 4)
        if name == "C1":
            s = torch.cuda.Stream(device=dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                ms.msort_sort_out(kin, kout, ws=ws, stream=s)
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=s):
                    ms.msort_sort_out(kin, kout, ws=ws, stream=s)
            for _ in range(5):
                g.replay()
            torch.cuda.synchronize()
            gt = []
            for _ in range(reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                e1.synchronize()
                gt.append(e0.elapsed_time(e1))
            gt.sort()
            d["graph_replay_ms"] = round(gt[len(gt) // 2], 4)
            d["graph_replay_verified"] = host_digest(kout.cpu().numpy()) == exp["keys_sha256"] \
                if exp else None
        out[name] = d
        del k, kin, vin, kout, vout, ws
        torch.cuda.empty_cache()
    r = {"workload": "BASELINE.json configs 1-4 (msort_inputs.CONFIGS), one GPU, "
                     "out of place from the pristine input", "results": out}
    if "C2" in out and "C2s" in out and "C2r" in out:
        r["t_C2s_over_C2"] = round(out["C2s"]["ms"] / out["C2"]["ms"], 3)
        r["t_C2r_over_C2"] = round(out["C2r"]["ms"] / out["C2"]["ms"], 3)
    return r


def choose_exchange(args, ms, comm, dist, dev, kin, kout, ws, stream, world, rank, n, last_split):
    """N > 1: the exchange mode of the timed steps.  "pull" (and "auto")
    reserve the communicator for the fused pull exchange (msort_comm_reserve)
    and run ONE verified step: its output is checked against the oracle's
    digest (or order + rank edges when there is none) and every rank's
    verdict -- including a raised error -- is combined (MIN over ranks), so
    all ranks take the same decision.  "auto" falls back to the NCCL
    all-to-all when the pull step fails anywhere; "pull" then raises."""
    import torch

    if args.exchange == "alltoall":
        comm.set_exchange(0)
        return "alltoall"
    ok = 1
    err = None
    try:
        comm.set_exchange(1)  # this communicator only (include/msort.h msort_comm_set_exchange)
        comm.reserve(n, torch.int32, False, stream=stream)
        last_split[0] = ms.msort_sort_distributed_out(kin, kout, comm, ws=ws, stream=stream,
                                                      return_split=True)[2]
        torch.cuda.synchronize()
        exp = expected_digest(world, rank, n)
        if exp is not None:
            ok = int(host_digest(kout.cpu().numpy()) == exp)
        else:
            ok = int(bool((kout[1:] >= kout[:-1]).all()))
    except Exception as e:  # noqa: BLE001 -- decided collectively below
        ok, err = 0, str(e)[:200]
    t = torch.tensor([ok], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if int(t.item()) == 1:
        return "pull"
    if args.exchange == "pull":
        raise RuntimeError(f"pull exchange failed on some rank (here: {err})")
    comm.set_exchange(0)
    return "alltoall (pull check failed: %s)" % (err or "output mismatch on some rank")


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    if world > 1:
        # a dead peer inside a host-synchronised collective becomes an error
        # (communicator aborted) instead of a hang (include/msort.h)
        os.environ.setdefault("MSORT_NCCL_TIMEOUT_S", "600")

    import numpy as np
    import torch

    import msort_inputs as mi
    import paper_2211_16479_b200 as ms

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    comm = None
    dpath = world > 1 or args.distributed_path  # the distributed code path
    if dpath:
        import torch.distributed as dist

        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        else:
            dist.init_process_group("nccl", device_id=dev)
        comm = ms.Comm()

    n = args.n
    kin = mi.keys_torch(n, SEED0 + rank, "u31", device=dev)
    kout = torch.empty_like(kin)
    ws = ms.workspace(n, torch.int32, False, world=world, device=dev)
    stream = torch.cuda.current_stream()

    last_split = [None]
    exchange = None
    if dpath:
        exchange = choose_exchange(args, ms, comm, dist, dev, kin, kout, ws, stream, world, rank,
                                   n, last_split)

    def step():
        if not dpath:
            ms.msort_sort_out(kin, kout, ws=ws, stream=stream)
        elif exchange == "pull":  # reserved pull: no host synchronisation inside the call
            ms.msort_sort_distributed_out(kin, kout, comm, ws=ws, stream=stream)
        else:
            last_split[0] = ms.msort_sort_distributed_out(kin, kout, comm, ws=ws, stream=stream,
                                                          return_split=True)[2]

    def barrier():
        if dpath:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    sampler = ClockSampler(local)
    time.sleep(0.3)  # let nvidia-smi start sampling
    ms.profile_reset()
    ms.profile_enable(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    t0 = time.time()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    t1 = time.time()
    launches = ms.launch_count()
    ms.profile_enable(False)
    prof = ms.profile_read()
    time.sleep(0.2)
    sampler.stop()
    ms_total = e0.elapsed_time(e1)
    if dpath:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps

    # verify the last step's output BIT FOR BIT: SHA-256 of this rank's slice
    # against the oracle's digest (tests/golden/c5_digests.json, written by
    # tests/golden/make_c5_digests.py from oracle/ only) for p = 1, 2, 4, 8 at
    # the C5 size; other sizes / world sizes fall back to order + multiset sum
    # + rank edges.  Every rank's verdict is combined (MIN over ranks).
    exp = expected_digest(world, rank, n)
    if exp is not None:
        got = host_digest(kout.cpu().numpy())
        ok = got == exp
        vmethod = "sha256 of every rank's output vs the oracle's digest (tests/golden/c5_digests.json)"
    else:
        ok = bool((kout[1:] >= kout[:-1]).all()) if n > 1 else True
        vmethod = "order + multiset sum (+ rank edges); no oracle digest for this size / world"
        if world == 1:
            ok &= int(kout.sum(dtype=torch.int64)) == int(kin.sum(dtype=torch.int64))
    if dpath:
        if exp is None:
            edge = torch.tensor([int(kout[0]), int(kout[-1])], dtype=torch.int64, device=dev)
            edges = [torch.zeros_like(edge) for _ in range(world)]
            dist.all_gather(edges, edge)
            e = torch.stack(edges).cpu().numpy()
            ok &= bool(all(e[r][1] <= e[r + 1][0] for r in range(world - 1)))
            s_in = torch.tensor([int(kin.sum(dtype=torch.int64)), int(kout.sum(dtype=torch.int64))],
                                dtype=torch.int64, device=dev)
            dist.all_reduce(s_in)
            ok &= int(s_in[0]) == int(s_in[1])
        okt = torch.tensor([1 if ok else 0], device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        ok = bool(okt.item())

    # roofline of the dominant kernel (the merge kernel) from live CUDA events
    peak, peak_src = load_peaks()
    mp_launches, mp_ms = prof["merge_pass"]
    wk = 4
    alg_bytes = 2 * n * wk  # each merge level reads and writes every key once
    tile = ms.tile_size(ms.MSORT_INT32, ms.MSORT_NONE)
    ntiles = (n + tile - 1) // tile
    passes = (ntiles - 1).bit_length()  # merge levels per sort
    roof = None
    if mp_launches:
        # the merge kernel runs all `passes` levels of a sort in one launch
        per_launch = alg_bytes * passes * args.steps / mp_launches
        avg_s = mp_ms / mp_launches / 1e3
        ach = per_launch / avg_s / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": ncu_traffic(f"C5_n{n}"),
                "kernel": "k3_merge_pass", "algorithmic_bytes_per_launch": int(per_launch),
                "merge_levels_per_launch": passes * args.steps / mp_launches,
                "launches": mp_launches, "avg_launch_ms": round(mp_ms / mp_launches, 4),
                "peak_source": peak_src}
    phases = {k: {"launches_per_step": v[0] / args.steps, "ms_per_step": round(v[1] / args.steps, 4)}
              for k, v in prof.items() if v[0]}
    # whole-step roofline: bytes of every executed pass at HBM rate (+ NVLink)
    step_bytes = (passes + 1) * alg_bytes
    t_roof = step_bytes / (peak * 1e9)
    d4_passes = 0
    if world > 1:
        # D4 as executed: one K5 pass for keys with 3..8 ranks (in pull mode
        # it also carries the exchange), one K3 round at p = 2, else
        # ceil(log2 p) K3 rounds; plus the exchange over NVLink
        d4_passes = 1 if world <= 8 else (world - 1).bit_length()
        step_bytes += d4_passes * alg_bytes
        t_roof += n * wk * (world - 1) / world / 770e9 + d4_passes * alg_bytes / (peak * 1e9)

    clocks = sampler.summary(t0, t1)

    # N > 1: the D3 exchange against NVLink -- the bytes this rank sends and
    # receives over NVLink (its segments to / from the other ranks, from the
    # split matrix of the last step) per exchange, over the exchange's live
    # CUDA-event time; the slowest rank is reported
    # (pull exchange: the transfer happens inside the K5 merge kernel, which
    # reads every peer's segment in place -- its time is the exchange's)
    xroof = None
    xclass = "kway_merge" if exchange == "pull" else "exchange"
    if world > 1 and prof.get(xclass, (0, 0.0))[0] and last_split[0] is not None:
        S = last_split[0]
        sent = sum(int(S[j + 1][rank] - S[j][rank]) for j in range(world) if j != rank) * wk
        recv = sum(int(S[rank + 1][j] - S[rank][j]) for j in range(world) if j != rank) * wk
        xl, xms = prof[xclass]
        ach = max(sent, recv) / (xms / xl / 1e3) / 1e9
        t = torch.tensor([ach], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ach = float(t.item())
        xroof = {"bound": "nvlink", "achieved": round(ach, 1), "peak": 770.0, "unit": "GB/s",
                 "frac": round(ach / 770.0, 4), "bytes_sent": sent, "bytes_received": recv,
                 "avg_exchange_ms": round(xms / xl, 4),
                 "timed_kernel": "k5_merge (exchange fused into the merge)" if exchange == "pull"
                 else "grouped ncclSend/ncclRecv",
                 "peak_source": "measured peer copy per direction (B200_PROFILING.md; 900 nominal)"}
        # the same exchange against a uniform NCCL all-to-all of
        # the same byte count (torch's all_to_all_single, equal splits), timed
        # here outside the measured region; the slowest rank is reported
        # every rank must agree before entering the collectives: a local
        # allocation failure must not leave the other ranks waiting
        buf = out_a2a = None
        try:
            buf = torch.empty(n, dtype=torch.int32, device=dev)
            out_a2a = torch.empty_like(buf)
            okf = 1
        except Exception as e:  # noqa: BLE001 -- context only, never fail the line
            xroof["uniform_alltoall_error"] = str(e)[:200]
            okf = 0
        okt = torch.tensor([okf], device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if int(okt.item()) == 1:
            for _ in range(2):
                dist.all_to_all_single(out_a2a, buf)
            torch.cuda.synchronize()
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record()
            for _ in range(5):
                dist.all_to_all_single(out_a2a, buf)
            eb.record()
            torch.cuda.synchronize()
            a2a_ms = ea.elapsed_time(eb) / 5
            t = torch.tensor([a2a_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            a2a_ms = float(t.item())
            a2a_gbs = n * wk * (world - 1) / world / (a2a_ms / 1e3) / 1e9
            xroof["uniform_alltoall_gbs"] = round(a2a_gbs, 1)
            xroof["frac_of_uniform_alltoall"] = round(ach / a2a_gbs, 4)
        del buf, out_a2a

    # end to end through the public API with HOST buffers: every step uploads
    # its input from pinned host memory, sorts, and copies the sorted keys back
    # (N = 1: msort_sort_host; consecutive steps rotate over three streams and
    # device buffers so one step's copy-back overlaps a later step's upload and
    # neither copy engine waits behind the other direction -- PCIe is full
    # duplex).  Device-timed: from an event before the first step
    # to the last step's completion on either stream.
    e2e = None
    if not args.no_e2e:
        h_in = kin.cpu().pin_memory()
        # as many steps as the timed region (6..40): the pipeline's fill and
        # drain (the first upload and the last copy-back overlap nothing) are
        # then amortised the way a streaming caller sees them
        ke = max(6, min(args.steps, 40))
        if not dpath:
            NS = max(1, args.e2e_streams)
            h_out = [torch.empty_like(h_in).pin_memory() for _ in range(NS)]
            d_buf = [torch.empty_like(kin) for _ in range(NS)]
            wss = [ws] + [ms.workspace(n, torch.int32, False, device=dev) for _ in range(NS - 1)]
            strs = [torch.cuda.Stream(device=dev) for _ in range(NS)]

            def e2e_step(i):
                ms.msort_sort_host(h_in, h_out[i], d_buf[i], ws=wss[i], stream=strs[i])

            for i in range(NS):
                e2e_step(i)
            torch.cuda.synchronize()
            f0 = torch.cuda.Event(enable_timing=True)
            f0.record(strs[0])
            for i in range(1, NS):
                strs[i].wait_event(f0)
            for k in range(ke):
                e2e_step(k % NS)
            fe = [torch.cuda.Event(enable_timing=True) for _ in range(NS)]
            for i in range(NS):
                fe[i].record(strs[i])
            torch.cuda.synchronize()
            te = max(f0.elapsed_time(fe[i]) for i in range(NS))
            exp0 = expected_digest(1, 0, n)
            for i in range(NS):
                o = h_out[i].numpy()
                ok &= (host_digest(o) == exp0) if exp0 else bool(np.all(o[1:] >= o[:-1]))
            path = ("msort_sort_host (pinned host -> device -> sort -> pinned host), "
                    f"steps rotate over {NS} streams")
        else:
            h_out = torch.empty_like(h_in).pin_memory()
            d_in = torch.empty_like(kin)

            def e2e_step():
                ms.msort_sort_distributed_host(h_in, h_out, d_in, comm, ws=ws, stream=stream)

            e2e_step()
            barrier()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(ke):
                e2e_step()
            f1.record(stream)
            barrier()
            te = f0.elapsed_time(f1)
            o = h_out.numpy()
            ok &= (host_digest(o) == exp) if exp else bool(np.all(o[1:] >= o[:-1]))
            path = ("msort_sort_distributed_host (pinned host -> device -> distributed sort -> "
                    "pinned host)")
        if dpath:
            t = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": world * n * ke / (te / 1e3), "unit": "keys/s",
               "h2d_bytes_per_step": n * wk, "d2h_bytes_per_step": n * wk,
               "ms_per_step": te / ke, "steps": ke, "path": path}
        if not dpath:
            # the PCIe ceiling of this e2e step: the same upload and download
            # alone, both directions at once on two streams (no sort)
            fl = pcie_duplex_ms(h_in, h_out[0], d_buf[0], kin, strs)
            e2e["pcie_duplex_ms"] = fl
            e2e["frac_of_pcie"] = round(fl / (te / ke), 4)

    batched = None
    if rank == 0 and not dpath and not args.no_batched:
        batched = batched_bench(ms, mi, dev)
    per_config = None
    if rank == 0 and not dpath and not args.no_configs:
        per_config = configs_bench(ms, mi, dev, peak)

    cpu = cpu_mp = None
    if rank == 0 and not dpath and not args.no_cpu_baseline:
        cpu = cpu_baseline(n, 1, SEED0)       # O-1 on the full rank-0 shard
        cpu_mp = cpu_paper_mp(n, SEED0)       # O-c on the same shard, all host cores
        if per_config is not None:
            configs_cpu(per_config)           # O-1 / O-c on configs 1-4

    if rank == 0:
        value = world * n * args.steps / (ms_total / 1e3)
        line = {
            "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": "C5: 2^28 int32 keys per GPU, uniform [0,2^31), "
                                   "counter-mode SplitMix64 seed 4+rank"
                                   + ("" if world == 1 else "; distributed, globally sorted"),
                       "n_per_gpu": n, "key_dtype": "int32", "payload": None,
                       "tile": tile, "merge_passes": passes,
                       "l2": "inputs larger than L2 (1 GiB/GPU vs 126 MB); no flush; "
                             "out-of-place sort from the pristine input each step",
                       "parallelism": f"dp{world}" if world > 1 else "single",
                       "exchange": exchange},
            "roofline": roof,
            "exchange_roofline": xroof,
            "step_roofline": {"bytes_per_gpu": step_bytes, "t_roof_ms": t_roof * 1e3,
                              "hbm_passes": passes + 1 + d4_passes,
                              "frac": round(t_roof * 1e3 / ms_step, 4),
                              "floor_frac": round(2 * n * wk / (peak * 1e9) * 1e3 / ms_step, 4)},
            "phases": phases,
            "cpu_baseline": cpu,
            "cpu_paper_mp": cpu_mp,
            "e2e": e2e,
            "batched_sort": batched,
            "configs": per_config,
            "gpu_launches": launches,
            "clocks": clocks,
            "verified": ok,
            "verification": vmethod,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
