"""Write tests/golden/oracle_golden.json from the CPU oracle ONLY.

Every stored expected value in tests/golden/ that is not the paper's own is
written by this script, which calls only `oracle/` and the seeded input
generator `msort_inputs` (no CUDA path).  Run:  python tests/golden/make_golden.py

The same quantities were computed independently with numpy during the survey
(SURVEY.md §8(c) "Golden values"); tests/test_oracle.py pins this file to those
independent numbers, which is what ties the oracle at full config size to
something other than itself.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import msort_inputs as mi  # noqa: E402
import oracle  # noqa: E402


def summary(name):
    k, v = mi.config_input(name)
    n = k.size
    out = {"n": n, "first_keys": k[:16].tolist(), "sum": int(k.astype(np.int64).sum()
                                                           if k.dtype != np.uint32 else
                                                           k.astype(np.uint64).sum())}
    if v is None:
        s = oracle.sort(k)
        pos = [0, n // 4, n // 2, 3 * n // 4, n - 1]
        out["sorted_at"] = {str(p): int(s[p]) for p in pos}
    else:
        s, sv = oracle.sort(k, v)
        pos = [0, 1, 2, n // 2, n - 1]
        out["sorted_at"] = {str(p): int(s[p]) for p in pos}
        out["payload_at"] = {str(p): int(sv[p]) for p in pos}
        out["check"] = oracle.check(k, s, sv)
    out["duplicates"] = int(n - 1 - int(np.count_nonzero(s[1:] != s[:-1])))
    return out


def main():
    g = {"_note": "written by tests/golden/make_golden.py from oracle/ only"}
    for name in ("C1", "C2", "C3", "C4"):
        g[name] = summary(name)
        print(name, g[name], flush=True)
    k = mi.keys(16, 2, ("mod", 1000))
    sk, sv = oracle.sort(k, mi.index_payload(16))
    g["C3_first16_sorted_pairs"] = [[int(a), int(b)] for a, b in zip(sk, sv)]
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_golden.json"), "w") as f:
        json.dump(g, f, indent=1)


if __name__ == "__main__":
    main()
