"""Random stress for the batched sort, the rank-tree gather and the K6 mode:
every case bit-exact to the oracle (seeded; sizes, length mixes, dtypes,
distributions and offsets location drawn at random)."""
import numpy as np
import pytest
import torch

import msort_inputs as mi

pytestmark = pytest.mark.gpu

from test_gpu_sort import _keys, check_parity, to_dev, to_host  # noqa: E402

DTS = [np.int32, np.uint32, np.int64, np.uint64]
DISTS = ["rand", "dup", "eq", "asc", "desc", "ext"]


@pytest.fixture(scope="module")
def ms():
    import paper_2211_16479_b200 as m

    assert torch.cuda.is_available()
    return m


def test_batched_random(ms, orc):
    rng = np.random.default_rng(1611)
    for t in range(40):
        nseg = int(rng.integers(1, 3000))
        scale = [4, 40, 400, 4000, 40000][int(rng.integers(0, 5))]
        lens = rng.integers(0, scale + 1, nseg)
        if rng.integers(0, 4) == 0:
            lens[int(rng.integers(0, nseg))] = int(rng.integers(0, 300000))  # one long segment
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        n = int(off[-1])
        dtype = DTS[int(rng.integers(0, 4))]
        k = _keys(n, 7000 + t, DISTS[int(rng.integers(0, len(DISTS)))], dtype)
        pairs = bool(rng.integers(0, 2))
        v = mi.index_payload(n) if pairs else None
        kd, vd = to_dev(k), (to_dev(v) if pairs else None)
        o = torch.from_numpy(off).cuda() if rng.integers(0, 2) else off
        ms.msort_sort_segmented(kd, o, vd)
        torch.cuda.synchronize()
        if pairs:
            ek, ev = orc.sort_segmented(k, off, v)
            assert np.array_equal(to_host(kd, dtype), ek), t
            assert np.array_equal(to_host(vd, np.uint32), ev), t
        else:
            assert np.array_equal(to_host(kd, dtype), orc.sort_segmented(k, off)), t


def test_tree_random(ms, orc):
    rng = np.random.default_rng(1612)
    for t in range(20):
        p = int(rng.integers(1, 12))
        dtype = DTS[int(rng.integers(0, 4))]
        dist = DISTS[int(rng.integers(0, len(DISTS)))]
        shards = [_keys(int(rng.integers(0, 50000)), 8000 + 16 * t + r, dist, dtype)
                  for r in range(p)]
        pairs = bool(rng.integers(0, 2))
        vals = ([((np.uint32(r) << np.uint32(24)) + np.arange(s.size, dtype=np.uint32))
                 for r, s in enumerate(shards)] if pairs else None)
        rk, rv = ms.msort_sort_distributed_tree_emulated(
            [to_dev(s) for s in shards], [to_dev(v) for v in vals] if pairs else None)
        torch.cuda.synchronize()
        exp = orc.sort_tree(shards, vals)
        if pairs:
            assert np.array_equal(to_host(rk, dtype), exp[0]), t
            assert np.array_equal(to_host(rv, np.uint32), exp[1]), t
        else:
            assert np.array_equal(to_host(rk, dtype), exp), t


def test_k6_random(ms, orc):
    ms.set_quad_mode(5)
    try:
        rng = np.random.default_rng(1613)
        for t in range(30):
            n = int(rng.integers(0, 1 << int(rng.integers(10, 23))))
            dtype = [np.int32, np.uint32][int(rng.integers(0, 2))]
            k = _keys(n, 9000 + t, DISTS[int(rng.integers(0, len(DISTS)))], dtype)
            check_parity(ms, orc, k, None)
    finally:
        ms.set_quad_mode(0)
