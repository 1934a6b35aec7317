"""GPU: the library is reentrant (include/msort.h, SURVEY §8(b) "Thread safety").

Host threads call the sorts at once, each on its own stream, in a FRESH
process -- so the first calls race through the lazy per-device set-up (kernel
attributes, grid sizes, the K0 cluster query, the memory pool) -- with
different dtypes, payloads and sizes (K0, K1 + fused K3, pairs); every result
is compared bit for bit with the oracle.
"""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import sys, threading
    sys.path.insert(0, %r)
    import numpy as np, torch
    import msort_inputs as mi, oracle
    import paper_2211_16479_b200 as ms

    NP = {"i32": np.int32, "u32": np.uint32, "i64": np.int64, "u64": np.uint64}
    TT = {"i32": torch.int32, "u32": torch.int32, "i64": torch.int64, "u64": torch.int64}
    jobs = []
    for t, (dist, n, pairs) in enumerate([
            ("i32", 50000, False), ("u32", 300000, False), ("i64", 1 << 20, False),
            ("u64", 70001, True), ("i32", (1 << 21) + 3, True), ("i64", 9000, True),
            ("u32", 1 << 16, False), ("i32", 5 * 8704 + 1, False)]):
        k = mi.keys(n, 3000 + t, dist)
        v = mi.index_payload(n) if pairs else None
        jobs.append((k, v))
    torch.cuda.init()
    errs, outs = [], [None] * len(jobs)

    def run(i):
        try:
            k, v = jobs[i]
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                kd = torch.from_numpy(k.view(np.int32 if k.itemsize == 4 else np.int64)).cuda()
                vd = torch.from_numpy(v.view(np.int32)).cuda() if v is not None else None
                for _ in range(2):  # the second sort re-sorts sorted data: same result
                    if vd is None:
                        ms.msort_sort(kd.view(torch.uint32) if k.dtype == np.uint32 else
                                      kd.view(torch.uint64) if k.dtype == np.uint64 else kd,
                                      stream=st)
                    else:
                        ms.msort_sort_pairs(kd.view(torch.uint32) if k.dtype == np.uint32 else
                                            kd.view(torch.uint64) if k.dtype == np.uint64 else kd,
                                            vd, stream=st)
                st.synchronize()
                outs[i] = (kd.cpu().numpy().view(k.dtype),
                           vd.cpu().numpy().view(np.uint32) if vd is not None else None)
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for (k, v), (ok, ov) in zip(jobs, outs):
        if v is None:
            assert np.array_equal(ok, oracle.sort(k)), "keys differ"
        else:
            ek, ev = oracle.sort(k, v)
            assert np.array_equal(ok, ek), "keys differ"
            assert np.array_equal(ov, ev), "payload differs"
    print("concurrent ok", len(jobs))
""") % ROOT


def test_concurrent_first_calls_fresh_process():
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "concurrent ok 8" in r.stdout
