"""Write tests/golden/config_digests.json from the CPU oracle ONLY.

For the single-GPU BASELINE.json configs C1-C4 (msort_inputs.config_input;
C3 and C4 carry the original index as payload): the
SHA-256 of the oracle's sorted keys and, for C3/C4, of the sorted payloads
(little-endian bytes), plus the first/last key.  bench.py's per-config lines
and the full-size GPU tests compare the GPU outputs against these digests,
i.e. bit for bit.  The oracle's full-size outputs of C1-C4 are pinned to the
survey's independent numpy values in tests/test_oracle.py (oracle_golden.json).

    python tests/golden/make_config_digests.py [--cores C]
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

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config_digests.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cores", type=int, default=len(os.sched_getaffinity(0)))
    a = ap.parse_args()
    out = {"_note": "written by tests/golden/make_config_digests.py from oracle/ only: SHA-256 of "
                    "the oracle's sorted keys (and payloads) of configs C1-C4", "configs": {}}
    t0 = time.time()
    for name in ("C1", "C2", "C3", "C4"):
        k, v = mi.config_input(name)
        k = k.copy()
        vv = None if v is None else v.copy()
        oracle.paper_mp_inplace(k, vv, a.cores)
        d = {"n": int(k.size), "dtype": str(k.dtype), "keys_sha256": sha(k), "first": int(k[0]),
             "last": int(k[-1])}
        if vv is not None:
            d["vals_sha256"] = sha(vv)
            d["vals_first"] = int(vv[0])
            d["vals_last"] = int(vv[-1])
        out["configs"][name] = d
        print(name, d, f"{time.time() - t0:.0f} s", flush=True)
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
