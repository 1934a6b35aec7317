"""GPU parity for the batched (segmented) sort, SURVEY.md §8(f) f3.

msort_sort_segmented through the C ABI vs the oracle's per-segment sort
(oracle.sort_segmented, pinned to numpy.lexsort in test_oracle.py), bit-exact.
Segment lengths cover every bin of Kernels::sort_segmented and its edges:
0/1 (no-ops), the warp bins (<= 32, <= 256), the CTA bins (<= 2176, <= the
tile T) and longer segments (the single-array sort), with duplicate-heavy keys
so stability is observable through the original-index payload.
"""
import numpy as np
import pytest
import torch

import msort_inputs as mi

pytestmark = pytest.mark.gpu

from test_gpu_sort import _keys, to_dev, to_host  # noqa: E402


@pytest.fixture(scope="module")
def ms():
    import paper_2211_16479_b200 as m

    assert torch.cuda.is_available()
    return m


def _run(ms, orc, k, off, pairs, dev_off=False):
    v = mi.index_payload(k.size) if pairs else None
    kd = to_dev(k)
    vd = to_dev(v) if pairs else None
    o = torch.as_tensor(np.asarray(off, dtype=np.int64)).cuda() if dev_off else off
    ms.msort_sort_segmented(kd, o, vd)
    torch.cuda.synchronize()
    if pairs:
        ek, ev = orc.sort_segmented(k, off, v)
        ok, ov = to_host(kd, k.dtype), to_host(vd, np.uint32)
        assert np.array_equal(ok, ek), f"keys differ at {np.nonzero(ok != ek)[0][:5]}"
        assert np.array_equal(ov, ev), f"payload differs at {np.nonzero(ov != ev)[0][:5]}"
    else:
        ek = orc.sort_segmented(k, off)
        ok = to_host(kd, k.dtype)
        assert np.array_equal(ok, ek), f"keys differ at {np.nonzero(ok != ek)[0][:5]}"


def _edges(ms, dtype, pairs):
    kd = {np.int32: ms.MSORT_INT32, np.uint32: ms.MSORT_UINT32, np.int64: ms.MSORT_INT64,
          np.uint64: ms.MSORT_UINT64}[dtype]
    T = ms.tile_size(kd, ms.MSORT_UINT32 if pairs else ms.MSORT_NONE)
    return [0, 1, 2, 3, 31, 32, 33, 100, 255, 256, 257, 1000, 2175, 2176, 2177, 4000, T - 1, T,
            T + 1, 2 * T + 5, 3 * T + 7, 0, 5]


@pytest.mark.parametrize("dtype", [np.int32, np.uint32, np.int64, np.uint64])
@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("dist", ["rand", "dup"])
@pytest.mark.parametrize("dev_off", [False, True])
def test_segment_bins(ms, orc, dtype, pairs, dist, dev_off):
    lens = _edges(ms, dtype, pairs)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    k = _keys(int(off[-1]), 11, dist, dtype)
    _run(ms, orc, k, off, pairs, dev_off)


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("dev_off", [False, True])
def test_many_small_segments(ms, orc, dtype, pairs, dev_off):
    """20000 segments of 0..300 elements (the warp bins, many CTAs of 4 warps)."""
    rng = np.random.default_rng(3)
    lens = rng.integers(0, 301, 20000)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    k = _keys(int(off[-1]), 12, "dup", dtype)
    _run(ms, orc, k, off, pairs, dev_off)


@pytest.mark.parametrize("dist", ["eq", "asc", "desc", "ext"])
def test_structured_segments(ms, orc, dist):
    rng = np.random.default_rng(5)
    lens = np.concatenate([rng.integers(0, 3000, 300), [20000]])
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    k = _keys(int(off[-1]), 13, dist, np.int32)
    _run(ms, orc, k, off, True)


def test_single_segment_is_plain_sort(ms, orc):
    n = (1 << 20) + 77
    k = mi.keys(n, 14, "i32")
    _run(ms, orc, k, [0, n], True)
    a = to_dev(k)
    b = to_dev(k)
    ms.msort_sort_segmented(a, [0, n])
    ms.msort_sort(b)
    assert torch.equal(a, b)


def test_segments_do_not_mix(ms):
    """Descending segment values: a sort that crossed a boundary would move
    keys between segments."""
    lens = [7, 300, 0, 1, 9000, 45]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    k = np.concatenate([np.full(l, 1000 - i, dtype=np.int32) - np.arange(l, dtype=np.int32) % 3
                        for i, l in enumerate(lens)])
    kd = to_dev(k)
    ms.msort_sort_segmented(kd, off)
    out = to_host(kd, np.int32)
    for i in range(len(lens)):
        a, b = off[i], off[i + 1]
        assert np.array_equal(np.sort(out[a:b]), np.sort(k[a:b]))
        assert np.all(out[a:b][1:] >= out[a:b][:-1])


def test_empty_and_invalid(ms):
    z = torch.empty(0, dtype=torch.int32, device="cuda")
    ms.msort_sort_segmented(z, [0])
    ms.msort_sort_segmented(z, [0, 0, 0])
    x = torch.arange(10, dtype=torch.int32, device="cuda")
    with pytest.raises(ms.MsortError):
        ms.msort_sort_segmented(x, [0, 6, 5, 10])
    with pytest.raises(ms.MsortError):
        ms.msort_sort_segmented(x, [0, 9])
    # device tables are checked on the device, before any key moves
    x0 = x.clone()
    for bad in ([0, 6, 5, 10], [0, 9], [1, 10], [0, 300, 0, 10]):
        with pytest.raises(ms.MsortError):
            ms.msort_sort_segmented(x, torch.tensor(bad, dtype=torch.int64, device="cuda"))
        assert torch.equal(x, x0)
    y = torch.randint(0, 1 << 30, (5000,), dtype=torch.int32, device="cuda")
    bad = torch.tensor([0] + [300, 0] * 20 + [5000], dtype=torch.int64, device="cuda")
    with pytest.raises(ms.MsortError):  # overlapping segments would overflow the lists
        ms.msort_sort_segmented(y, bad)


@pytest.mark.parametrize("dtype", [np.int32, np.uint32, np.int64])
@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("dev_off", [False, True])
def test_many_long_segments(ms, orc, dtype, pairs, dev_off):
    """Segments longer than a tile with 1..6 merge levels (both buffer
    parities) mixed with short ones: one fused merge launch over all of them."""
    rng = np.random.default_rng(21)
    lens = np.concatenate([rng.integers(8705, 60000, 150), rng.integers(0, 9000, 150),
                           [17 * 8704 + 3, 40 * 8704, 5 * 8704, 2]])
    rng.shuffle(lens)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    k = _keys(int(off[-1]), 22, "dup" if pairs else "rand", dtype)
    _run(ms, orc, k, off, pairs, dev_off)


def test_segmented_repeat_and_streams(ms, orc):
    """Back-to-back calls reuse the staging buffer (the second call's tables
    must not overwrite the first's before they reach the device)."""
    rng = np.random.default_rng(31)
    outs = []
    s2 = torch.cuda.Stream()
    for it in range(4):
        lens = rng.integers(0, 20000, 200)
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        k = _keys(int(off[-1]), 40 + it, "rand", np.int32)
        kd = to_dev(k)
        torch.cuda.synchronize()
        ms.msort_sort_segmented(kd, off, stream=s2 if it % 2 else None)
        outs.append((k, off, kd))
    torch.cuda.synchronize()
    for k, off, kd in outs:
        assert np.array_equal(to_host(kd, np.int32), orc.sort_segmented(k, off))


def test_segmented_concurrent_host_threads(ms, orc):
    """Host threads calling the batched sort at once on their own streams share
    the page-locked staging buffer (a mutex and an upload event order them);
    every result must be its own table's."""
    import threading

    rng = np.random.default_rng(77)
    jobs = []
    for t in range(8):
        lens = rng.integers(0, 12000, 150)
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        k = _keys(int(off[-1]), 900 + t, "rand", np.int32)
        jobs.append((k, off, to_dev(k), torch.cuda.Stream()))
    torch.cuda.synchronize()
    errs = []

    def run(job):
        k, off, kd, st = job
        try:
            for _ in range(3):  # re-sorting sorted segments is idempotent
                ms.msort_sort_segmented(kd, off, stream=st)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(j,)) for j in jobs]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errs, errs
    for k, off, kd, _ in jobs:
        assert np.array_equal(to_host(kd, np.int32), orc.sort_segmented(k, off))


@pytest.mark.parametrize("pairs", [False, True])
def test_long_host_table(ms, orc, pairs):
    """A host table of >= 2^15 segments is uploaded and classified on the device
    (Kernels::sort_segmented); mixed lengths so every bin is used."""
    rng = np.random.default_rng(41)
    lens = rng.integers(0, 40, 100000)
    lens[rng.integers(0, lens.size, 30)] = rng.integers(300, 30000, 30)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    k = _keys(int(off[-1]), 42, "dup", np.int32)
    _run(ms, orc, k, off, pairs, dev_off=False)
