"""Workspace bounds: every call that takes a caller workspace gets EXACTLY the
size msort_*workspace_bytes reports, carved from a larger buffer whose tail is
a canary; the sort must be right and the canary untouched (no write past the
reported size), for the length distributions that stress each part of the
carve-up (segment lists, K1 tile descriptors, merge counters, K6 tables)."""
import numpy as np
import pytest
import torch

import msort_inputs as mi

pytestmark = pytest.mark.gpu

from test_gpu_sort import to_dev, to_host  # noqa: E402

CANARY = 1 << 20


@pytest.fixture(scope="module")
def ms():
    import paper_2211_16479_b200 as m

    assert torch.cuda.is_available()
    return m


def _ws(nbytes):
    nbytes = (nbytes + 255) // 256 * 256
    buf = torch.full((nbytes + CANARY,), 0xA5, dtype=torch.uint8, device="cuda")
    return buf, buf[:nbytes]


def _canary_ok(buf, nbytes):
    nbytes = (nbytes + 255) // 256 * 256
    return bool((buf[nbytes:] == 0xA5).all())


@pytest.mark.parametrize("shape", ["all33", "all257", "all2177", "allTp1", "giant", "tiny2",
                                   "mixed"])
@pytest.mark.parametrize("dev_off", [False, True])
@pytest.mark.parametrize("pairs", [False, True])
def test_segmented_workspace_exact(ms, orc, shape, dev_off, pairs):
    T = ms.tile_size(ms.MSORT_INT32, ms.MSORT_UINT32 if pairs else ms.MSORT_NONE)
    n = 1 << 20
    L = {"all33": 33, "all257": 257, "all2177": 2177, "allTp1": T + 1, "giant": n,
         "tiny2": 2}.get(shape)
    if L is not None:
        lens = np.full(n // L, L)
        lens = np.append(lens, n - lens.sum()) if lens.sum() < n else lens
    else:
        lens = np.random.default_rng(2).integers(0, 3 * T, 2000)
        lens = lens[: np.searchsorted(np.cumsum(lens), n)]
        lens = np.append(lens, n - lens.sum())
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    k = mi.keys(n, 7, ("mod", 1000)).astype(np.int32)
    v = mi.index_payload(n)
    kd, vd = to_dev(k), (to_dev(v) if pairs else None)
    nb = ms.msort_segmented_workspace_bytes(n, off.size - 1, ms.MSORT_INT32,
                                           ms.MSORT_UINT32 if pairs else ms.MSORT_NONE)
    buf, ws = _ws(nb)
    o = torch.from_numpy(off).cuda() if dev_off else off
    ms.msort_sort_segmented(kd, o, vd, ws=ws)
    torch.cuda.synchronize()
    assert _canary_ok(buf, nb), "segmented sort wrote past its workspace"
    if pairs:
        ek, ev = orc.sort_segmented(k, off, v)
        assert np.array_equal(to_host(kd, np.int32), ek)
        assert np.array_equal(to_host(vd, np.uint32), ev)
    else:
        assert np.array_equal(to_host(kd, np.int32), orc.sort_segmented(k, off))


@pytest.mark.parametrize("mode", [0, 5])
@pytest.mark.parametrize("n", [8704 * 4 + 1, (1 << 22) + 5])
def test_sort_workspace_exact(ms, orc, mode, n):
    ms.set_quad_mode(mode)
    try:
        k = mi.keys(n, 8, "i32")
        kin, kout = to_dev(k), torch.empty(n, dtype=torch.int32, device="cuda")
        nb = ms.msort_workspace_bytes(n, ms.MSORT_INT32)
        buf, ws = _ws(nb)
        ms.msort_sort_out(kin, kout, ws=ws)
        torch.cuda.synchronize()
        assert _canary_ok(buf, nb)
        assert np.array_equal(to_host(kout, np.int32), orc.sort(k))
    finally:
        ms.set_quad_mode(0)


@pytest.mark.parametrize("span", [1000, 1 << 40])  # key-range narrowed / the 8-byte path
@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("n", [65537, (1 << 21) + 3])
def test_sort_workspace_exact_int64(ms, orc, span, pairs, n):
    """8-byte keys with exactly the reported workspace: both enqueued paths
    (one gated off on the device) and the range slot stay inside it."""
    rng = np.random.default_rng(n + span)
    k = (rng.integers(0, span, n, dtype=np.int64) - span // 2).astype(np.int64)
    v = mi.index_payload(n) if pairs else None
    kin = to_dev(k)
    kout = torch.empty_like(kin)
    vin = to_dev(v) if pairs else None
    vout = torch.empty_like(vin) if pairs else None
    nb = ms.msort_workspace_bytes(n, ms.MSORT_INT64, ms.MSORT_UINT32 if pairs else ms.MSORT_NONE)
    buf, ws = _ws(nb)
    ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
    torch.cuda.synchronize()
    assert _canary_ok(buf, nb), "8-byte sort wrote past its workspace"
    if pairs:
        ek, ev = orc.sort(k, v)
        assert np.array_equal(to_host(kout, np.int64), ek)
        assert np.array_equal(to_host(vout, np.uint32), ev)
    else:
        assert np.array_equal(to_host(kout, np.int64), orc.sort(k))
