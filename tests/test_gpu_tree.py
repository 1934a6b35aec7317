"""GPU parity for the paper's rank-tree gather (SURVEY.md §8(f) f4,
include/msort.h msort_sort_distributed_tree): rank 0's result vs the oracle's
literal run of the paper's loop (oracle.sort_tree, pinned in
test_oracle.py), bit-exact, for p virtual ranks on one GPU (device copies in
place of NCCL send/recv) and the real NCCL path with one rank.
"""
import os

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


def _shards(p, sizes, dtype, dist, seed):
    out = []
    for r in range(p):
        out.append(_keys(int(sizes[r]), seed + r, dist, dtype))
    return out


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("dtype,pairs", [(np.int32, False), (np.int32, True), (np.uint64, True),
                                         (np.int64, False)])
def test_tree_emulated(ms, orc, p, dtype, pairs):
    rng = np.random.default_rng(100 + p)
    sizes = rng.integers(0, 60000, p)
    sizes[p // 2] = 0 if p > 2 else sizes[p // 2]  # an empty rank
    shards = _shards(p, sizes, dtype, "dup", 50)
    vals = ([((np.uint32(r) << np.uint32(24)) + np.arange(s.size, dtype=np.uint32))
             for r, s in enumerate(shards)] if pairs else None)
    kd = [to_dev(s) for s in shards]
    vd = [to_dev(v) for v in vals] if pairs else None
    rk, rv = ms.msort_sort_distributed_tree_emulated(kd, vd)
    torch.cuda.synchronize()
    exp = orc.sort_tree(shards, vals)
    if pairs:
        assert np.array_equal(to_host(rk, dtype), exp[0])
        assert np.array_equal(to_host(rv, np.uint32), exp[1])
    else:
        assert np.array_equal(to_host(rk, dtype), exp)
    # the inputs are read only
    for s, d in zip(shards, kd):
        assert np.array_equal(to_host(d, dtype), s)


def test_tree_c5_shape(ms, orc):
    """C5-shaped shards (2^22 int32 per rank here, seed 4 + r) at p = 8: the root
    holds the sorted concatenation; payload = (rank, index) in tree order."""
    p, n = 8, 1 << 22
    shards = [mi.keys(n, 4 + r, "i32") for r in range(p)]
    vals = [((np.uint32(r) << np.uint32(28)) + np.arange(n, dtype=np.uint32)) for r in range(p)]
    rk, rv = ms.msort_sort_distributed_tree_emulated([to_dev(s) for s in shards],
                                                     [to_dev(v) for v in vals])
    torch.cuda.synchronize()
    order = orc.tree_rank_order(p)
    cat = np.concatenate([shards[r] for r in order])
    catv = np.concatenate([vals[r] for r in order])
    ek = cat.copy()
    ev = catv.copy()
    orc.paper_mp_inplace(ek, ev, os.cpu_count() or 1)
    assert np.array_equal(to_host(rk, np.int32), ek)
    assert np.array_equal(to_host(rv, np.uint32), ev)


def test_tree_nccl_one_rank(ms, orc):
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    comm = ms.Comm()
    n = 70001
    k = mi.keys(n, 78, ("mod", 50))
    v = np.arange(n, dtype=np.uint32)
    rk, rv = ms.msort_sort_distributed_tree(to_dev(k), comm, in_vals=to_dev(v))
    torch.cuda.synchronize()
    ek, ev = orc.sort(k, v)
    assert np.array_equal(to_host(rk, np.int64), ek)
    assert np.array_equal(to_host(rv, np.uint32), ev)
    comm.close()
