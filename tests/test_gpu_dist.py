"""GPU parity of the distributed path (D1-D4) on one B200.

Multi-rank: the library's single-process emulation runs p virtual ranks on
one device with the same kernels, splitter planning and k-way merge (the
NCCL calls replaced by device reductions/copies).  The real NCCL path runs at
p = 1 with a one-rank communicator.  Expected values: oracle.split_matrix and
oracle slices of the stably sorted rank-major concatenation (R10/R11),
plus the independent C5 split matrices of SURVEY.md §8(c) addendum.
"""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import msort_inputs as mi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[0, 1], ids=["alltoall", "pull"])
def ms(request):
    """Every test runs with both exchange modes (include/msort.h
    msort_debug_set_exchange): NCCL-style all-to-all + k-way merge, and the
    fused pull (the first merge round reads the peers' segments in place)."""
    import paper_2211_16479_b200 as m

    m.set_exchange_mode(request.param)
    yield m
    m.set_exchange_mode(0)


def _dev(a):
    if a.dtype == np.uint32:
        return torch.from_numpy(a.view(np.int32)).cuda().view(torch.uint32)
    if a.dtype == np.uint64:
        return torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    return torch.from_numpy(a).cuda()


def _host(t, dt):
    if t.dtype == torch.uint32:
        t = t.view(torch.int32)
    if t.dtype == torch.uint64:
        t = t.view(torch.int64)
    return t.cpu().numpy().view(dt)


def run_emulated(ms, orc, shards, pairs):
    p = len(shards)
    K = np.concatenate([[0], np.cumsum([s.size for s in shards])])
    vals = [np.arange(K[r], K[r + 1], dtype=np.uint32) for r in range(p)] if pairs else None
    kd = [_dev(s) for s in shards]
    vd = [_dev(v) for v in vals] if pairs else None
    split = ms.msort_sort_distributed_emulated(kd, vd)
    torch.cuda.synchronize()
    assert np.array_equal(split, orc.split_matrix(shards))
    cat = np.concatenate(shards)
    if pairs:
        ek, ev = orc.sort(cat, np.arange(cat.size, dtype=np.uint32))
    else:
        ek, ev = orc.sort(cat), None
    for r in range(p):
        assert np.array_equal(_host(kd[r], cat.dtype), ek[K[r]:K[r + 1]]), f"rank {r} keys"
        if pairs:
            assert np.array_equal(_host(vd[r], np.uint32), ev[K[r]:K[r + 1]]), f"rank {r} vals"


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 7, 8])
@pytest.mark.parametrize("pairs", [False, True])
def test_emulated_random_unequal_sizes(ms, orc, p, pairs):
    rng = np.random.default_rng(p * 10 + pairs)
    for trial in range(3):
        sizes = rng.integers(0, 40000, size=p)
        if trial == 1:
            sizes[0] = 0
        if trial == 2 and p > 2:
            sizes[p // 2] = 0
            sizes[-1] = 1
        shards = [mi.keys(int(s), 1000 * p + 10 * trial + r, "i32") for r, s in enumerate(sizes)]
        run_emulated(ms, orc, shards, pairs)


@pytest.mark.parametrize("p", [3, 5, 8])
def test_emulated_skewed_ranges(ms, orc, p):
    """Rank j holds keys only in [ (p-1-j) 2^20, (p-j) 2^20 ) (reversed rank
    order) or all in one narrow band: every rank's output comes from one or
    two source ranks, so the K5 runs are extremely unequal (most empty) --
    the device-planned K5 of the pull exchange and the received-run K5 of
    the all-to-all both see it."""
    shards = []
    for r in range(p):
        z = mi.splitmix64(30000 + 1000 * r, 700 + r) % np.uint64(1 << 20)
        shards.append((z.astype(np.int64) + ((p - 1 - r) << 20)).astype(np.int32))
    run_emulated(ms, orc, shards, False)
    band = [(mi.splitmix64(25000, 800 + r) % np.uint64(64)).astype(np.int32) + 7 for r in range(p)]
    band[1] = band[1][:0]  # and an empty rank
    run_emulated(ms, orc, band, False)


@pytest.mark.parametrize("dtype,dist", [(np.int64, ("mod", 5)), (np.uint32, "eq"),
                                        (np.int32, "eq"), (np.uint64, "u64"),
                                        (np.int64, ("mod", 1000))])
def test_emulated_duplicates_across_ranks(ms, orc, dtype, dist):
    """Keys equal across shards: ties must be handed out in rank order."""
    for p in (2, 3, 8):
        sizes = [9000 + 1000 * r for r in range(p)]
        if dist == "eq":
            shards = [np.full(s, 7, dtype=dtype) for s in sizes]
        elif dist == "u64":
            shards = [mi.keys(s, 50 + r, "u64") for r, s in enumerate(sizes)]
        else:
            shards = [mi.keys(s, 60 + r, dist).astype(dtype) for r, s in enumerate(sizes)]
        run_emulated(ms, orc, shards, True)


def test_emulated_extremes(ms, orc):
    for dtype in (np.int32, np.uint32, np.int64, np.uint64):
        info = np.iinfo(dtype)
        pool = np.array([info.min, 0, info.max], dtype=dtype)
        shards = [pool[(mi.splitmix64(5000 + r, r) % np.uint64(3)).astype(np.int64)]
                  for r in range(4)]
        run_emulated(ms, orc, shards, True)


# SURVEY.md §8(c) addendum: C5 split rows (independent numpy computation)
C5_ROWS = {
    2: {1: [134212162, 134223294]},
    4: {1: [67110172, 67108539, 67110135, 67106610],
        2: [134217801, 134228923, 134215104, 134209084],
        3: [201323646, 201329812, 201327789, 201325121]},
    8: {1: [33556935, 33554878, 33558649, 33554402, 33564042, 33547661, 33550740, 33548149],
        4: [134219922, 134230981, 134217240, 134211196, 134216455, 134211743, 134221324,
            134212963],
        7: [234880444, 234882874, 234877251, 234874288, 234885948, 234884604, 234881155,
            234881628]},
}


def _c5_digests():
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                           "c5_digests.json")) as f:
        return json.load(f)["digests"]


def _sha(t):
    a = t.cpu().numpy()
    return hashlib.sha256(a.view(np.uint8)).hexdigest()


@pytest.mark.parametrize("p", [2, 4, 8])
def test_c5_full_size_bit_exact(ms, p):
    """C5 at full size (2^28 int32 per rank, seed 4+rank), emulated p ranks (in
    both exchange modes, module fixture): the split matrix equals the survey's, and EVERY rank's
    output equals the oracle's expected slice byte for byte (SHA-256 against
    tests/golden/c5_digests.json, written from oracle/ only)."""
    n = 1 << 28
    dig = _c5_digests()[str(p)]
    kd = [mi.keys_torch(n, 4 + r, "u31", device="cuda") for r in range(p)]
    split = ms.msort_sort_distributed_emulated(kd)
    torch.cuda.synchronize()
    for r, row in C5_ROWS[p].items():
        assert split[r].tolist() == row
    for r, k in enumerate(kd):
        assert _sha(k) == dig[r]["sha256"], f"rank {r} of {p}"
    del kd
    torch.cuda.empty_cache()


def test_c5_single_gpu_bit_exact(ms):
    """The one-GPU C5 sort (bench.py's workload) equals the oracle's sorted
    shard byte for byte (SHA-256 digest, p = 1 row)."""
    n = 1 << 28
    kin = mi.keys_torch(n, 4, "u31", device="cuda")
    kout = torch.empty_like(kin)
    ms.msort_sort_out(kin, kout)
    torch.cuda.synchronize()
    assert _sha(kout) == _c5_digests()["1"][0]["sha256"]
    del kin, kout
    torch.cuda.empty_cache()


def test_nccl_one_rank(ms, orc):
    """The real NCCL path with a one-rank communicator on this GPU."""
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    comm = ms.Comm()
    n = 100003
    k = mi.keys(n, 77, ("mod", 100))
    v = np.arange(n, dtype=np.uint32)
    kd, vd = _dev(k), _dev(v)
    _, _, split = ms.msort_sort_distributed(kd, comm, vals=vd, return_split=True)
    torch.cuda.synchronize()
    ek, ev = orc.sort(k, v)
    assert split.tolist() == [[0], [n]]
    assert np.array_equal(_host(kd, np.int64), ek)
    assert np.array_equal(_host(vd, np.uint32), ev)
    comm.close()


def test_nccl_one_rank_reserve_pull(ms, orc):
    """msort_comm_reserve on the real NCCL communicator (one rank): the
    exchange buffer is allocated and published through CUDA IPC, the device
    shard table written; pull-mode sorts within the reservation are exact
    (at one rank the call is the local sort; the multi-GPU test covers the
    reserved K5 path)."""
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    comm = ms.Comm()
    n = 70001
    comm.reserve(n)
    comm.set_exchange(1)  # per communicator (the process default stays 0)
    try:
        for seed in (1, 2):
            k = mi.keys(n - seed, 80 + seed, "i32")
            kd = _dev(k)
            ms.msort_sort_distributed(kd, comm)
            torch.cuda.synchronize()
            assert np.array_equal(_host(kd, np.int32), orc.sort(k))
        comm.set_exchange(-1)  # back to the process default
        k = mi.keys(n, 83, "i32")
        kd = _dev(k)
        ms.msort_sort_distributed(kd, comm)
        torch.cuda.synchronize()
        assert np.array_equal(_host(kd, np.int32), orc.sort(k))
        with pytest.raises(ms.MsortError):
            comm.set_exchange(2)
    finally:
        comm.close()


def test_nccl_one_rank_host_buffers(ms, orc):
    """msort_sort_distributed_host (bench.py's N > 1 e2e path) on the one-rank
    NCCL communicator: pinned host keys in, the sorted slice back in host
    memory."""
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    comm = ms.Comm()
    n = 123457
    k = mi.keys(n, 91, "i32")
    h_in = torch.from_numpy(k.copy()).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    ms.msort_sort_distributed_host(h_in, h_out, d, comm)
    torch.cuda.synchronize()
    assert np.array_equal(h_out.numpy(), orc.sort(k))
    assert np.array_equal(h_in.numpy(), k)
    comm.close()


def test_nccl_wait_timeout_aborts(tmp_path):
    """Failure detection (include/msort.h): with MSORT_NCCL_TIMEOUT_S set, a
    distributed call whose stream does not drain in time (here: held up by a
    1 s sleep kernel, standing in for a dead peer) returns MSORT_ERROR_NCCL,
    aborts the communicator, and later calls on it fail at once.  (With one
    rank the balanced sort needs no host wait, so the rank-tree call -- which
    always waits for the shard sizes -- is the one that can be held up.)"""
    import subprocess
    import sys

    code = r'''
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
import paper_2211_16479_b200 as ms
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29541", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
comm = ms.Comm()
k = torch.randint(0, 1000, (1 << 16,), dtype=torch.int32, device="cuda")
s2 = torch.cuda.Stream()
with torch.cuda.stream(s2):
    torch.cuda._sleep(2_000_000_000)  # ~1 s on the call's stream
try:
    ms.msort_sort_distributed_tree(k, comm, stream=s2)
    print("NO-ERROR")
except ms.MsortError as e:
    print("ERR1", "timed out" in str(e))
try:
    ms.msort_sort_distributed_tree(k, comm, stream=s2)
    print("NO-ERROR2")
except ms.MsortError as e:
    print("ERR2", "aborted" in str(e))
torch.cuda.synchronize()
comm.close()
'''
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MSORT_NCCL_TIMEOUT_S="0.05", ROOT=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=240)
    assert "ERR1 True" in r.stdout and "ERR2 True" in r.stdout, r.stdout + r.stderr[-2000:]


def test_comm_wrap_torch(ms, orc):
    """msort_comm_wrap: the library runs the distributed sort (and the tree)
    on torch's own NCCL communicator; closing the wrapper leaves torch's
    process group usable."""
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    comm = ms.Comm.from_torch()
    assert (comm.rank, comm.world) == (0, 1)
    n = 90001
    k = mi.keys(n, 79, ("mod", 77))
    v = np.arange(n, dtype=np.uint32)
    kd, vd = _dev(k), _dev(v)
    ms.msort_sort_distributed(kd, comm, vals=vd)
    rk, _ = ms.msort_sort_distributed_tree(_dev(k), comm)
    torch.cuda.synchronize()
    ek, ev = orc.sort(k, v)
    assert np.array_equal(_host(kd, np.int64), ek)
    assert np.array_equal(_host(vd, np.uint32), ev)
    assert np.array_equal(_host(rk, np.int64), ek)
    comm.close()
    t = torch.ones(1, device="cuda")
    dist.all_reduce(t)  # torch's communicator still works
    assert float(t.item()) == 1.0


def test_python_layer_calls(ms, orc):
    """SURVEY §8(b) Python layer: sort (clone), sort_ (in place), sort_pairs,
    sort_distributed (in place, cached communicator)."""
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    n = 30011
    k = mi.keys(n, 81, ("mod", 500))
    v = np.arange(n, dtype=np.uint32)
    kd = _dev(k)
    out = ms.sort(kd)
    assert np.array_equal(_host(out, np.int64), orc.sort(k))
    assert np.array_equal(_host(kd, np.int64), k)  # unchanged
    ms.sort_(kd)
    assert np.array_equal(_host(kd, np.int64), orc.sort(k))
    sk, sv = ms.sort_pairs(_dev(k), _dev(v))
    ek, ev = orc.sort(k, v)
    assert np.array_equal(_host(sk, np.int64), ek) and np.array_equal(_host(sv, np.uint32), ev)
    kd2, vd2 = _dev(k), _dev(v)
    for _ in range(2):  # second call reuses the cached communicator
        kk, vv = ms.sort_distributed(kd2, vals=vd2)
    torch.cuda.synchronize()
    assert np.array_equal(_host(kk, np.int64), ek) and np.array_equal(_host(vv, np.uint32), ev)
