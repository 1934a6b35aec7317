"""GPU parity of the K6 4-way merge pass (keys only) against the CPU oracle.

msort_debug_set_quad(5) runs every pair of merge levels as one K6 pass (unit
tiles between X-side states, cut at Y-side states, merged with the tile
sort's engine), so small inputs (many groups, ragged groups, cuts) go
through it; mode 0 (2-way levels only) must give the identical result.
Every expected value comes from oracle/ on the same seeded input.  (The K3Q
and K3X experiments are no longer built: experiments/*.cuh.txt.)
"""
import numpy as np
import pytest
import torch

import msort_inputs as mi

from test_gpu_sort import _keys, gpu_sort, oracle_sort, to_dev, to_host

pytestmark = pytest.mark.gpu

DTYPES = [np.int32, np.uint32, np.int64, np.uint64]


@pytest.fixture(scope="module", params=[5], ids=["k6"])
def ms(request):
    """Mode 5: K6 (unit tiles between X-side states, cut at Y-side states,
    merged with the tile-sort engine; 4-byte keys -- 8-byte keys take mode 0)."""
    import paper_2211_16479_b200 as m

    assert torch.cuda.is_available()
    m.set_quad_mode(request.param)
    m.QUAD_TEST_MODE = request.param
    yield m
    m.set_quad_mode(0)


def _check(ms, orc, k):
    ok, _ = gpu_sort(ms, k, None)
    ek, _ = oracle_sort(orc, k, None)
    bad = np.nonzero(ok != ek)[0]
    assert bad.size == 0, f"n={k.size} keys differ at {bad[:5]} (of {bad.size})"


@pytest.mark.parametrize("dtype", DTYPES)
def test_quad_sizes(ms, orc, dtype):
    kd = {np.int32: 0, np.uint32: 1, np.int64: 2, np.uint64: 3}[dtype]
    T = ms.tile_size(kd, ms.MSORT_NONE)
    # 2 levels (one 4-way pass), 3 (4-way + 2-way), 4, 5, 6 levels; ragged groups
    sizes = [3 * T + 1, 4 * T, 4 * T + 7, 7 * T - 5, 16 * T, 16 * T + 3, 33 * T + 1000,
             64 * T - 1, 200003, 300001, 1 << 20]
    for i, n in enumerate(sizes):
        for dist in ("rand", "dup"):
            _check(ms, orc, _keys(n, 300 + i, dist, dtype))


@pytest.mark.parametrize("dist", ["eq", "asc", "desc", "ext", "dup"])
@pytest.mark.parametrize("dtype", DTYPES)
def test_quad_structured(ms, orc, dist, dtype):
    """All-equal keys (one tie block split across segments by rank-order
    fill), sorted / reversed runs (one input of a node used up first), the
    dtype's extremes (real maximum keys tie with the used-up sentinels)."""
    for n in (5 * 8704 * 4 + 77, 600001):
        _check(ms, orc, _keys(n, 9, dist, dtype))


def test_quad_max_keys_everywhere(ms, orc):
    """Half the keys are the maximum int32: every node meets sentinel ties."""
    n = 400000
    k = mi.keys(n, 21, "i32")
    k[::2] = np.iinfo(np.int32).max
    _check(ms, orc, k)
    k = np.full(n, np.iinfo(np.uint32).max, dtype=np.uint32)
    k[:1000] = 7
    _check(ms, orc, k)


def test_quad_modes_agree(ms):
    """Modes 0 / 5 sort a 2^22 shard to the same bytes."""
    n = 1 << 22
    src = mi.keys_torch(n, 5, "u31", device="cuda")
    outs = []
    for mode in (0, 5):
        ms.set_quad_mode(mode)
        t = src.clone()
        ms.msort_sort(t)
        outs.append(t)
    ms.set_quad_mode(ms.QUAD_TEST_MODE)
    torch.cuda.synchronize()
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    assert bool((outs[0][1:] >= outs[0][:-1]).all())


def test_quad_out_of_place_misaligned(ms, orc):
    """Out-of-place sort from / to views that are not 16-byte aligned: the
    rings keep each window's global 16-byte phase."""
    n = 250000
    for off in (1, 3):
        base = mi.keys(n + off, 40 + off, "i32")
        kin = to_dev(base)[off:]
        kout = torch.empty(n + 4, dtype=torch.int32, device="cuda")[off:off + n]
        ws = ms.workspace(n, torch.int32, False, device="cuda")
        ms.msort_sort_out(kin, kout, ws=ws)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(kout, np.int32), orc.sort(base[off:].copy()))
