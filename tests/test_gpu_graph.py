"""CUDA graph capture of the sort (include/msort.h: the workspace calls are
asynchronous, allocation-free and synchronisation-free, so a stream capture
records memset + K1 + the fused K3 and a replay sorts whatever the input
buffer holds).  Checked bit-exactly against the oracle on new data per replay."""
import numpy as np
import pytest
import torch

import msort_inputs as mi

pytestmark = pytest.mark.gpu

from test_gpu_sort import to_dev, to_host  # noqa: E402


@pytest.fixture(scope="module")
def ms():
    import paper_2211_16479_b200 as m

    assert torch.cuda.is_available()
    return m


@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("n", [(1 << 16) + 3, 1 << 20])
def test_graph_replay(ms, orc, pairs, n):
    kin = torch.empty(n, dtype=torch.int32, device="cuda")
    kout = torch.empty_like(kin)
    vin = torch.empty(n, dtype=torch.int32, device="cuda") if pairs else None
    vout = torch.empty_like(vin) if pairs else None
    ws = ms.workspace(n, torch.int32, pairs, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up (one-time kernel attribute setup) outside the capture
        ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
    for seed in (1, 2, 3):
        k = mi.keys(n, 60 + seed, ("mod", 1000) if pairs else "i32").astype(np.int32)
        v = mi.index_payload(n)
        kin.copy_(to_dev(k))
        if pairs:
            vin.copy_(to_dev(v).view(torch.int32))
        g.replay()
        torch.cuda.synchronize()
        if pairs:
            ek, ev = orc.sort(k, v)
            assert np.array_equal(to_host(kout, np.int32), ek)
            assert np.array_equal(to_host(vout, np.int32).view(np.uint32), ev)
        else:
            assert np.array_equal(to_host(kout, np.int32), orc.sort(k))


@pytest.mark.parametrize("pairs", [False, True])
def test_graph_replay_int64_range_decided_on_device(ms, orc, pairs):
    """One captured 8-byte-key sort serves both key-range paths: the choice
    between the narrowed (32-bit offsets) and the 8-byte sort is taken on the
    device at every replay, so replays alternate between narrow-range and
    full-range inputs and each is bit-exact."""
    n = (1 << 20) + 77
    kin = torch.zeros(n, dtype=torch.int64, device="cuda")
    kout = torch.empty_like(kin)
    vin = torch.empty(n, dtype=torch.int32, device="cuda") if pairs else None
    vout = torch.empty_like(vin) if pairs else None
    ws = ms.workspace(n, torch.int64, pairs, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
    v = mi.index_payload(n)
    for i, span in enumerate([1000, 1 << 62, (1 << 32) - 1, 1 << 32]):
        rng = np.random.default_rng(100 + i)
        k = (rng.integers(0, span, n, dtype=np.int64) - (1 << 61)).astype(np.int64)
        kin.copy_(to_dev(k))
        if pairs:
            vin.copy_(to_dev(v).view(torch.int32))
        g.replay()
        torch.cuda.synchronize()
        if pairs:
            ek, ev = orc.sort(k, v)
            assert np.array_equal(to_host(kout, np.int64), ek)
            assert np.array_equal(to_host(vout, np.uint32), ev)
        else:
            assert np.array_equal(to_host(kout, np.int64), orc.sort(k))
