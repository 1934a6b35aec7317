"""GPU: sorts larger than 2^31 elements (64-bit indexing everywhere: tile
indices, co-ranks, byte offsets) -- keys only and with a uint32 payload.

The oracle cannot sort 2^31 keys in test time, so these checks are properties
that hold at any size and pin the result: the output is
non-decreasing; it is the input multiset (sum and sum of squares mod 2^64);
sampled output positions p satisfy #{x < out[p]} <= p < #{x <= out[p]} over
the input -- the counting-rank definition of the sorted sequence; with a
payload of original indices, the payload is a permutation, out_keys ==
in_keys[payload], and equal keys keep increasing indices (stability).
"""
import pytest
import torch

import msort_inputs as mi

pytestmark = pytest.mark.gpu

N_LARGE = (1 << 31) + 12345


@pytest.fixture(scope="module")
def ms():
    import paper_2211_16479_b200 as m

    assert torch.cuda.is_available()
    return m


def _multiset(t: torch.Tensor):
    x = t.to(torch.int64)  # sums wrap mod 2^64
    return int(x.sum()), int((x * x).sum()), int((x ^ (x >> 17)).sum())


def _check_keys(kin: torch.Tensor, kout: torch.Tensor, seed: int):
    assert bool((kout[1:] >= kout[:-1]).all()), "not non-decreasing"
    assert _multiset(kin) == _multiset(kout), "not the input multiset"
    g = torch.Generator().manual_seed(seed)
    n = kin.numel()
    for p in [0, n - 1] + torch.randint(0, n, (6,), generator=g).tolist():
        v = kout[p]
        lt = int((kin < v).sum())
        le = int((kin <= v).sum())
        assert lt <= p < le, f"position {p}: {lt} <= {p} < {le} fails"


@pytest.mark.parametrize("dist", ["u31", "i64"])
def test_keys_beyond_2g(ms, dist):
    kin = mi.keys_torch(N_LARGE, 31, dist, device="cuda")
    kout = torch.empty_like(kin)
    ms.msort_sort_out(kin, kout)
    torch.cuda.synchronize()
    _check_keys(kin, kout, 1)


def test_pairs_beyond_2g(ms):
    n = N_LARGE
    kin = mi.keys_torch(n, 32, "u31", device="cuda")
    # many ties: keys in [0, 2^20) so stability is exercised everywhere
    kin >>= 11
    idx = torch.arange(n, dtype=torch.int64, device="cuda").to(torch.int32)  # uint32 bits
    k = kin.clone()
    v = idx.clone().view(torch.uint32)
    ms.msort_sort_pairs(k, v)
    torch.cuda.synchronize()
    _check_keys(kin, k, 2)
    vi = v.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    mark = torch.zeros(n, dtype=torch.bool, device="cuda")
    mark[vi] = True
    assert bool(mark.all()), "payload is not a permutation"
    del mark
    assert torch.equal(kin[vi], k), "out_keys != in_keys[payload]"
    eq = k[1:] == k[:-1]
    assert bool((vi[1:][eq] > vi[:-1][eq]).all()), "equal keys out of original order"
