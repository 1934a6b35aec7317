"""CPU-side checks of the C-ABI library (no GPU): it loads, exports every
symbol include/msort.h declares, validates arguments before touching the
device, and its host-side splitter planning reproduces the oracle's split
matrix."""
import ctypes
import os
import re

import numpy as np
import pytest

import msort_inputs as mi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ms():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2211_16479_b200 as m

    return m


def test_exports_every_declared_symbol(ms):
    with open(os.path.join(ROOT, "include", "msort.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"\b(msort_[a-z0-9_]+)\s*\(", hdr))
    declared -= {"msort_stream_t"}
    assert len(declared) >= 20
    for name in sorted(declared):
        assert hasattr(ms.lib, name), name  # ctypes resolves the symbol
    assert set(ms.EXPORTED) == declared


def test_validation_without_device(ms):
    L = ms.lib
    assert L.msort_sort(None, 0, 0, None) == 0
    assert L.msort_sort(None, 1, 0, None) == 1  # NULL with n > 0
    assert L.msort_sort(ctypes.c_void_p(4096), 10, 9, None) == 1  # unknown dtype
    assert L.msort_sort(ctypes.c_void_p(4098), 10, 0, None) == 1  # misaligned
    assert L.msort_sort(ctypes.c_void_p(4096), (1 << 40) + 1, 0, None) == 1
    assert L.msort_sort_pairs(ctypes.c_void_p(4096), ctypes.c_void_p(4100), 10, 0, 1, None) == 1
    assert L.msort_sort_pairs(ctypes.c_void_p(4096), ctypes.c_void_p(1 << 20), 10, 0, 2, None) == 2
    assert L.msort_sort_pairs(ctypes.c_void_p(4096), None, 10, 0, 255, None) == 1
    assert ms.lib.msort_status_string(5) == b"MSORT_ERROR_NCCL"
    out = ctypes.c_size_t()
    assert L.msort_workspace_bytes(1 << 20, 0, 255, 1, ctypes.byref(out)) == 0
    assert out.value >= (1 << 20) * 4
    # segmented sort: offsets must start at 0, not decrease and end at n
    S = L.msort_sort_segmented
    bad = (ctypes.c_int64 * 3)(0, 5, 4)
    assert S(ctypes.c_void_p(4096), None, 4, bad, 2, 0, 255, None, 0, None) == 1
    bad2 = (ctypes.c_int64 * 3)(1, 2, 4)
    assert S(ctypes.c_void_p(4096), None, 4, bad2, 2, 0, 255, None, 0, None) == 1
    assert S(ctypes.c_void_p(4096), None, 4, None, 2, 0, 255, None, 0, None) == 1
    ok0 = (ctypes.c_int64 * 1)(0)
    assert S(None, None, 0, ok0, 0, 0, 255, None, 0, None) == 0
    sb = ctypes.c_size_t()
    assert L.msort_segmented_workspace_bytes(1 << 20, 1000, 0, 1, ctypes.byref(sb)) == 0
    assert sb.value >= 16 * 1000
    n2 = ctypes.c_size_t()
    assert L.msort_workspace_bytes(1 << 20, 2, 1, 8, ctypes.byref(n2)) == 0
    assert n2.value >= 2 * (1 << 20) * 12


def test_plan_constants(ms):
    assert ms.plan_rounds(ms.MSORT_INT32) == 4 and ms.plan_rounds(ms.MSORT_UINT64) == 8
    assert ms.plan_candidates_per_round() == 256
    lohi = ms.plan_init(ms.MSORT_INT32, 3)
    assert lohi.tolist() == [0, 0xFFFFFFFF, 0, 0xFFFFFFFF]
    c = ms.plan_candidates(3, lohi)
    assert c.shape == (2, 256) and int(c[0, -1]) == 0xFFFFFFFF and int(c[0, 0]) == (1 << 24) - 1
    assert (np.diff(c[0].astype(np.int64)) > 0).all()


IMAGE = {np.int32: lambda a: a.view(np.uint32) ^ np.uint32(0x80000000),
         np.uint32: lambda a: a,
         np.int64: lambda a: a.view(np.uint64) ^ np.uint64(1 << 63),
         np.uint64: lambda a: a}
KD = {np.int32: 0, np.uint32: 1, np.int64: 2, np.uint64: 3}


def plan_split(ms, shards):
    """Run the host planning functions over p in-process shards (the counts a
    GPU count kernel would produce, taken here with numpy searchsorted)."""
    p = len(shards)
    dt = shards[0].dtype.type
    imgs = [np.sort(IMAGE[dt](s)) for s in shards]
    K = np.concatenate([[0], np.cumsum([s.size for s in shards])]).astype(np.uint64)
    lohi = ms.plan_init(KD[dt], p)
    for _ in range(ms.plan_rounds(KD[dt])):
        cand = ms.plan_candidates(p, lohi)
        total = sum(np.searchsorted(im, cand.ravel(), side="right").astype(np.uint64)
                    for im in imgs)
        lohi = ms.plan_narrow(p, K, total, lohi)
    v = lohi[0::2]
    assert np.array_equal(lohi[0::2], lohi[1::2])  # converged to a single image
    lteq = np.zeros((p, p - 1, 2), dtype=np.uint64)
    for j, im in enumerate(imgs):
        lt = np.searchsorted(im, v, side="left")
        le = np.searchsorted(im, v, side="right")
        lteq[j, :, 0], lteq[j, :, 1] = lt, le - lt
    return ms.plan_fill(p, K, lteq)


def test_plan_matches_oracle_split_matrix(ms, orc):
    rng = np.random.default_rng(3)
    for trial in range(120):
        p = int(rng.integers(1, 9))
        dt = [np.int32, np.uint32, np.int64, np.uint64][trial % 4]
        sizes = rng.integers(0, 300, size=p)
        if trial % 5 == 0:
            sizes[rng.integers(0, p)] = 0
        mode = trial % 3
        shards = []
        for r, s in enumerate(sizes):
            s = int(s)
            if mode == 0:
                a = mi.keys(s, trial * 10 + r, {np.int32: "i32", np.uint32: "u32",
                                                 np.int64: "i64", np.uint64: "u64"}[dt])
            elif mode == 1:
                a = mi.keys(s, trial * 10 + r, ("mod", 4)).astype(dt)
            else:
                info = np.iinfo(dt)
                pool = np.array([info.min, 0, info.max], dtype=dt)
                a = pool[(mi.splitmix64(s, r) % np.uint64(3)).astype(np.int64)]
            shards.append(np.asarray(a, dtype=dt))
        got = plan_split(ms, shards)
        assert np.array_equal(got, orc.split_matrix(shards)), (trial, sizes)
