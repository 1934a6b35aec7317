"""GPU parity of the p-way merge (include/msort.h msort_merge_runs; K5 for keys
with 3..16 runs, K3 rounds otherwise) against the CPU oracle.

The expected output is the oracle's stable sort of the concatenated runs with
the global index as payload (ties: lower run, then lower index -- merge() of
P:107 generalised, R1/R11).  The run layouts stress the K5 tile
partition: empty runs, one run much longer than the others, runs that cover
disjoint key ranges (every tile draws from one run), all-equal keys across
runs (one tie block cut at sample boundaries), the dtype's extreme keys (real
keys equal to the MIN/MAX sentinels), odd run lengths (windows at every
16-byte phase), and sizes around the tile capacity.
"""
import numpy as np
import pytest
import torch

import msort_inputs as mi

from test_gpu_sort import to_dev, to_host

pytestmark = pytest.mark.gpu

DTYPES = [np.int32, np.uint32, np.int64, np.uint64]
DIST = {np.int32: "i32", np.uint32: "u32", np.int64: "i64", np.uint64: "u64"}


@pytest.fixture(scope="module")
def ms():
    """K5 takes up to 16 runs here (MSORT_K5=16; the product default is 8,
    above which K3 rounds are faster), so every K5 shape is exercised."""
    import os

    import paper_2211_16479_b200 as m

    assert torch.cuda.is_available()
    old = os.environ.get("MSORT_K5")
    os.environ["MSORT_K5"] = "16"
    yield m
    if old is None:
        os.environ.pop("MSORT_K5", None)
    else:
        os.environ["MSORT_K5"] = old


def _dev(a):
    return to_dev(np.ascontiguousarray(a))


def _host(t, dtype):
    return to_host(t, dtype)


def _runs(sizes, seed, dtype, kind="rand"):
    out = []
    for j, s in enumerate(sizes):
        if kind == "rand":
            k = mi.keys(s, seed + j, DIST[dtype]).astype(dtype)
        elif kind == "dup":
            k = (mi.splitmix64(s, seed + j) % np.uint64(7)).astype(dtype)
        elif kind == "eq":
            k = np.full(s, 5, dtype=dtype)
        elif kind == "ext":
            info = np.iinfo(dtype)
            pool = np.array([info.min, info.min, 0, info.max, info.max], dtype=dtype)
            k = pool[(mi.splitmix64(s, seed + j) % np.uint64(5)).astype(np.int64)]
        elif kind == "disjoint":  # run j holds keys in [j*2^20, (j+1)*2^20), reversed run order
            base = (len(sizes) - 1 - j) << 20
            k = (base + (mi.splitmix64(s, seed + j) % np.uint64(1 << 20)).astype(np.int64)).astype(dtype)
        else:
            raise ValueError(kind)
        out.append(np.sort(k, kind="stable"))
    return out


def _check(ms, orc, runs, pairs=False):
    dtype = runs[0].dtype
    off = np.concatenate([[0], np.cumsum([r.size for r in runs])]).astype(np.int64)
    cat = np.concatenate(runs) if off[-1] else np.zeros(0, dtype=dtype)
    n = cat.size
    idx = np.arange(n, dtype=np.uint32)
    ek, ev = orc.sort(cat, idx)
    kin = _dev(cat)
    vin = _dev(idx) if pairs else None
    ko, vo = ms.msort_merge_runs(kin, off, in_vals=vin)
    torch.cuda.synchronize()
    got = _host(ko, dtype)
    bad = np.nonzero(got != ek)[0]
    assert bad.size == 0, f"p={len(runs)} n={n}: keys differ at {bad[:5]} (of {bad.size})"
    if pairs:
        assert np.array_equal(_host(vo, np.uint32), ev), f"p={len(runs)}: payload differs"
    assert np.array_equal(_host(kin, dtype), cat), "input modified"


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("p", [2, 3, 4, 5, 7, 8, 9, 12, 16])
def test_merge_random_unequal(ms, orc, dtype, p):
    sizes = [3000 + 7919 * ((j * 5) % p) + (j % 3) for j in range(p)]
    _check(ms, orc, _runs(sizes, 10 + p, dtype))


@pytest.mark.parametrize("kind", ["dup", "eq", "ext", "disjoint"])
@pytest.mark.parametrize("dtype", DTYPES)
def test_merge_structured(ms, orc, kind, dtype):
    for p in (3, 8, 16):
        sizes = [20000 + 1001 * j for j in range(p)]
        _check(ms, orc, _runs(sizes, 40, dtype, kind))


@pytest.mark.parametrize("p", [3, 4, 8, 16])
def test_merge_empty_and_skewed_runs(ms, orc, p):
    for sizes in ([0] * (p - 1) + [50000],          # one non-empty run (last)
                  [50000] + [0] * (p - 1),          # one non-empty run (first)
                  [0, 1] + [0] * (p - 3) + [2],     # almost nothing
                  [200000] + [3] * (p - 1),         # one giant run
                  [1] * p):
        _check(ms, orc, _runs(sizes, 77, np.int32))
    _check(ms, orc, _runs([0] * p, 1, np.int32))  # all empty


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_merge_tile_capacity_edges(ms, orc, dtype):
    """Sizes around the tile capacity and sample stride, all 16-byte phases."""
    for p in (3, 8):
        for base in (8000, 8431, 8432, 8433, 17000):
            sizes = [base + j for j in range(p)]
            _check(ms, orc, _runs(sizes, base, dtype))


def test_merge_large(ms, orc):
    """2^24 keys in 8 runs (the C5 shape at p = 8, scaled) and 16 runs."""
    for p in (8, 16):
        sizes = [(1 << 24) // p + 13 * j for j in range(p)]
        _check(ms, orc, _runs(sizes, 5, np.int32))


@pytest.mark.parametrize("p", [2, 3, 8, 17, 33])
def test_merge_pairs_and_many_runs(ms, orc, p):
    """With a payload (K3 rounds) and beyond 16 runs (K3 rounds): same bytes
    as the oracle, stable by run then index."""
    sizes = [1000 + 37 * j for j in range(p)]
    _check(ms, orc, _runs(sizes, 3, np.int32, "dup"), pairs=True)
    _check(ms, orc, _runs(sizes, 4, np.int64, "dup"), pairs=False)


def test_merge_argument_errors(ms):
    k = torch.arange(10, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        ms.msort_merge_runs(k, [0, 5, 9])  # does not end at n
    with pytest.raises(ms.MsortError):
        ms.msort_merge_runs(k, [0, 6, 5, 10])  # decreasing
    with pytest.raises(ms.MsortError):
        ms.msort_merge_runs(k, [0, 5, 10], keys_out=k)  # in place: overlap
