"""The multi-process path on CPU: world_size 2 (and 3) over torch.distributed
`gloo`, one process per rank, as bench.py runs under torchrun.

Each rank runs the distributed protocol of msort_sort_distributed with the
library's own host-side planning (msort_plan_* -- the arithmetic the K4
kernels run) and real collectives over gloo: the candidate counts are
all-reduced, (lt, eq) all-gathered, the split matrix filled, the sorted
segments exchanged point to point (D3) and merged (D4).  Local sorting,
counting and merging use the CPU oracle / numpy as stand-ins for the GPU
kernels.  Checked: every rank computes the same split matrix, it equals the
oracle's, and rank r ends with the oracle slice [K_r, K_{r+1}).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

IMAGE = {np.dtype(np.int32): lambda a: a.view(np.uint32) ^ np.uint32(0x80000000),
         np.dtype(np.uint32): lambda a: a,
         np.dtype(np.int64): lambda a: a.view(np.uint64) ^ np.uint64(1 << 63),
         np.dtype(np.uint64): lambda a: a}
KD = {np.dtype(np.int32): 0, np.dtype(np.uint32): 1, np.dtype(np.int64): 2, np.dtype(np.uint64): 3}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_shard(case, rank):
    import msort_inputs as mi

    sizes, dist_, dtype = case
    n = sizes[rank]
    if dist_ == "eq":
        return np.full(n, 3, dtype=dtype)
    return mi.keys(n, 4 + rank, dist_).astype(dtype)


def _worker(rank, world, port, cases, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch

    import oracle
    import paper_2211_16479_b200 as ms

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        for ci, case in enumerate(cases):
            shard = make_shard(case, rank)
            dt = shard.dtype
            kd = KD[dt]
            # D1: local sort (oracle stands in for K1..K3)
            local = oracle.sort(shard) if shard.size else shard.copy()
            img = IMAGE[dt](local)
            # sizes -> K
            nsz = torch.zeros(world, dtype=torch.int64)
            dist.all_gather_into_tensor(nsz, torch.tensor([local.size], dtype=torch.int64))
            K = np.concatenate([[0], np.cumsum(nsz.numpy())]).astype(np.uint64)
            # D2: bucket search rounds with all-reduced counts
            lohi = ms.plan_init(kd, world)
            for _ in range(ms.plan_rounds(kd)):
                cand = ms.plan_candidates(world, lohi)
                le = np.searchsorted(img, cand.ravel(), side="right").astype(np.int64)
                t = torch.from_numpy(le)
                dist.all_reduce(t)
                lohi = ms.plan_narrow(world, K, t.numpy().astype(np.uint64), lohi)
            v = lohi[0::2]
            lt = np.searchsorted(img, v, side="left")
            le = np.searchsorted(img, v, side="right")
            mine = np.stack([lt, le - lt], axis=1).astype(np.int64).ravel()
            allc = torch.zeros(world * mine.size, dtype=torch.int64)
            dist.all_gather_into_tensor(allc, torch.from_numpy(mine))
            S = ms.plan_fill(world, K, allc.numpy().astype(np.uint64))
            # D3: exchange the segments point to point
            reqs, recv = [], {}
            for j in range(world):
                if j == rank:
                    continue
                seg = local[S[j, rank]:S[j + 1, rank]]
                cnt = S[rank + 1, j] - S[rank, j]
                if seg.size:
                    reqs.append(dist.isend(torch.from_numpy(seg.view(np.int64) if dt.itemsize == 8
                                                            else seg.view(np.int32)).clone(), j))
                if cnt:
                    buf = torch.empty(int(cnt), dtype=torch.int64 if dt.itemsize == 8 else torch.int32)
                    recv[j] = buf
                    reqs.append(dist.irecv(buf, j))
            for r_ in reqs:
                r_.wait()
            runs = []
            for j in range(world):
                if j == rank:
                    runs.append(local[S[rank, rank]:S[rank + 1, rank]])
                elif j in recv:
                    runs.append(recv[j].numpy().view(dt))
                else:
                    runs.append(local[:0])
            # D4: stable k-way merge, lower source rank first (oracle merge rounds)
            while len(runs) > 1:
                nxt = []
                for m in range(0, len(runs), 2):
                    nxt.append(oracle.merge(runs[m], runs[m + 1]) if m + 1 < len(runs)
                               else runs[m])
                runs = nxt
            out = runs[0]
            q.put((ci, rank, S.tolist(), out.tobytes(), str(dt)))
    finally:
        dist.destroy_process_group()


CASES = [
    ([40000, 25000], "u31", np.int32),
    ([0, 30000], "i32", np.int32),
    ([1000, 1000], ("mod", 7), np.int64),
    ([5000, 7000], "eq", np.uint32),
    ([3000, 2000], "u64", np.uint64),
    ([1, 0], "i64", np.int64),
]
CASES3 = [
    ([10000, 0, 20000], "u31", np.int32),
    ([4000, 5000, 6000], ("mod", 3), np.int64),
]


def _run(world, cases, orc):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world * len(cases)):
        ci, rank, S, out, dt = q.get(timeout=300)
        got[(ci, rank)] = (np.array(S), np.frombuffer(out, dtype=np.dtype(dt)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, case in enumerate(cases):
        shards = [make_shard(case, r) for r in range(world)]
        ref_S = orc.split_matrix(shards)
        cat = np.concatenate(shards)
        ref = orc.sort(cat)
        K = np.concatenate([[0], np.cumsum([s.size for s in shards])])
        for r in range(world):
            S, out = got[(ci, r)]
            assert np.array_equal(S, ref_S), (ci, r)
            assert np.array_equal(out, ref[K[r]:K[r + 1]]), (ci, r)


def test_gloo_world2(orc):
    _run(2, CASES, orc)


def test_gloo_world3(orc):
    _run(3, CASES3, orc)


# ---------------------------------------------------------------- rank tree
def _tree_worker(rank, world, port, cases, q):
    """The rank-tree gather (msort_sort_distributed_tree) on CPU: the library's
    own schedule (msort_plan_tree_role), arrays moved point to point over
    gloo (sizes first), merged by the oracle's merge() as the stand-in for K3,
    local sorts by the oracle."""
    import sys

    sys.path.insert(0, ROOT)
    import torch

    import oracle
    import paper_2211_16479_b200 as ms

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        for ci, case in enumerate(cases):
            k = make_shard(case, rank)
            v = ((np.uint32(rank) << np.uint32(24)) + np.arange(k.size, dtype=np.uint32))
            k, v = oracle.sort(k, v)
            for role, peer in ms.plan_tree(world, rank):
                if role == 2:  # child: size, keys, payload to the parent
                    dist.send(torch.tensor([k.size], dtype=torch.int64), peer)
                    if k.size:
                        dist.send(torch.from_numpy(k.copy()), peer)
                        dist.send(torch.from_numpy(v.view(np.int32).copy()), peer)
                elif role == 1:  # parent: receive, merge(own, received)
                    m = torch.zeros(1, dtype=torch.int64)
                    dist.recv(m, peer)
                    m = int(m.item())
                    if m:
                        rk = torch.from_numpy(np.zeros(m, dtype=k.dtype))
                        rv = torch.zeros(m, dtype=torch.int32)
                        dist.recv(rk, peer)
                        dist.recv(rv, peer)
                        k, v = oracle.merge(k, rk.numpy(), v, rv.numpy().view(np.uint32))
            q.put((ci, rank, k.tobytes() if rank == 0 else b"", v.tobytes() if rank == 0 else b"",
                   k.dtype.str))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_gloo_tree(orc, world):
    cases = [([1000 * (r + 1) for r in range(world)], ("mod", 5), np.int64),
             ([0] + [777] * (world - 1), "u31", np.int32)]
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tree_worker, args=(r, world, port, cases, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world * len(cases)):
        ci, rank, kb, vb, dt = q.get(timeout=300)
        got[(ci, rank)] = (kb, vb, dt)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, case in enumerate(cases):
        shards = [make_shard(case, r) for r in range(world)]
        vals = [((np.uint32(r) << np.uint32(24)) + np.arange(s.size, dtype=np.uint32))
                for r, s in enumerate(shards)]
        ek, ev = orc.sort_tree(shards, vals)
        kb, vb, dt = got[(ci, 0)]
        assert np.array_equal(np.frombuffer(kb, dtype=np.dtype(dt)), ek)
        assert np.array_equal(np.frombuffer(vb, dtype=np.uint32), ev)


@pytest.fixture(scope="module")
def ms():
    import sys

    sys.path.insert(0, ROOT)
    import paper_2211_16479_b200 as m

    return m


def test_plan_tree_schedule(ms):
    """Every round pairs each child with exactly one parent; after the rounds
    only rank 0 holds data; powers of two follow the paper's split = size/2."""
    for p in range(1, 20):
        holds = set(range(p))
        rounds = ms.lib.msort_plan_tree_rounds(p)
        assert rounds == (p - 1).bit_length()
        for t in range(rounds):
            roles = [ms.plan_tree(p, r)[t] for r in range(p)]
            parents = {r: peer for r, (role, peer) in enumerate(roles) if role == 1}
            children = {r: peer for r, (role, peer) in enumerate(roles) if role == 2}
            assert {c: par for par, c in parents.items()} == children
            assert set(children) <= holds
            holds -= set(children)
            if p & (p - 1) == 0:  # the paper's split = size / 2^(t+1)
                split = p >> (t + 1)
                assert all(par == c - split for c, par in children.items())
        assert holds == {0}
