"""Write tests/golden/c5_digests.json from the CPU oracle ONLY.

The C5 workload (BASELINE.json config 5; SURVEY.md §8(c) "Distributed
oracle"): rank r holds 2^28 int32 keys uniform in [0, 2^31), counter-mode
SplitMix64 seed 4 + r (msort_inputs).  The distributed sort's expected output
on rank r of a p-rank run is the slice [r * 2^28, (r + 1) * 2^28) of the
stable sort of the rank-major concatenation (readings R10/R11).

This script computes that slice for p = 1, 2, 4, 8 with the oracle only:
every shard sorted by the paper's multiprocessing merge sort re-created on
host threads (oracle.paper_mp_inplace, pinned equal to the textbook
msort_oracle_sort in tests/test_oracle.py), then the shards merged pairwise by
the oracle's merge() (ties to the left run) -- SURVEY §8(c) allows
"oracle_sort on each shard, then a textbook p-way merge".  For keys only the
pairwise merge tree gives the same array as the rank-order p-way merge.

Stored per (p, r): the SHA-256 of the slice's little-endian bytes, its first
and last key and its int64 sum -- bench.py (`verified`) and the full-size GPU
tests compare every rank's output against the digest, i.e. bit for bit.

    python tests/golden/make_c5_digests.py [--cores C]      (~16 GB of host RAM)
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import msort_inputs as mi  # noqa: E402
import oracle  # noqa: E402

N = 1 << 28
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c5_digests.json")


def digest(a: np.ndarray) -> dict:
    a = np.ascontiguousarray(a, dtype="<i4")
    return {"sha256": hashlib.sha256(a.view(np.uint8)).hexdigest(), "first": int(a[0]),
            "last": int(a[-1]), "sum": int(a.astype(np.int64).sum())}


def slices(m: np.ndarray, p: int) -> list:
    return [digest(m[r * N:(r + 1) * N]) for r in range(p)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cores", type=int, default=len(os.sched_getaffinity(0)))
    a = ap.parse_args()
    t0 = time.time()
    s = []
    for r in range(8):
        k = mi.keys(N, 4 + r, "u31")
        oracle.paper_mp_inplace(k, None, a.cores)
        s.append(k)
        print(f"shard {r} sorted ({time.time() - t0:.0f} s)", flush=True)
    out = {"_note": "written by tests/golden/make_c5_digests.py from oracle/ only: per-rank "
                    "expected outputs of the C5 distributed sort (2^28 int32 keys per rank, "
                    "seed 4+rank), SHA-256 of the little-endian slice bytes",
           "n_per_rank": N, "digests": {}}
    out["digests"]["1"] = [digest(s[0])]
    m01 = oracle.merge(s[0], s[1])
    out["digests"]["2"] = slices(m01, 2)
    m23 = oracle.merge(s[2], s[3])
    m0123 = oracle.merge(m01, m23)
    del m01, m23
    out["digests"]["4"] = slices(m0123, 4)
    m45 = oracle.merge(s[4], s[5])
    m67 = oracle.merge(s[6], s[7])
    del s
    m4567 = oracle.merge(m45, m67)
    del m45, m67
    mall = oracle.merge(m0123, m4567)
    del m0123, m4567
    out["digests"]["8"] = slices(mall, 8)
    out["seconds"] = round(time.time() - t0, 1)
    out["cores"] = a.cores
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["digests"]["2"]), flush=True)


if __name__ == "__main__":
    main()
