"""The distributed path over REAL NCCL across >= 2 GPUs (one process per GPU).

Runs only where torch sees at least two GPUs (skipped on the one-GPU gpurun
boxes, where the single-process emulation in test_gpu_dist.py covers the same
kernels and planning).  Each worker process drives one GPU through
msort_sort_distributed / msort_sort_distributed_tree over a torch NCCL group
and checks its own output against the oracle on the same seeded shards, which
every worker regenerates:

  * the balanced sort (D1-D4), both exchange modes (NCCL all-to-all + k-way
    merge, and the pull exchange), keys only and with a uint32 payload,
    unequal shard sizes with an EMPTY rank, keys duplicated across ranks,
    int32 and int64 keys: rank r's output must equal the slice
    [K_r, K_r + n_r) of the oracle's stable sort of the rank-major
    concatenation (R10/R11), and the split matrix must equal
    oracle.split_matrix;
  * the rank-tree gather (the paper's loop): rank 0's output must
    equal oracle.sort_tree;
  * the same balanced sort on torch's own communicator (msort_comm_wrap).

Workers report through files; any mismatch fails the test with its text.
"""
import json
import os
import socket
import traceback

import numpy as np
import pytest
import torch

import msort_inputs as mi

pytestmark = pytest.mark.gpu

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shards(p, case):
    """Every worker builds the same shards: (keys list, vals list or None)."""
    if case == "unequal":
        sizes = [0 if r == 1 else 20000 + 7919 * r for r in range(p)]
        ks = [mi.keys(s, 500 + r, ("mod", 300)).astype(np.int32) for r, s in enumerate(sizes)]
    elif case == "int64":
        sizes = [50000 + 1000 * r for r in range(p)]
        ks = [mi.keys(s, 600 + r, "i64") for r, s in enumerate(sizes)]
    else:  # "equal": C5-shaped keys (uniform [0, 2^31)), equal sizes
        ks = [mi.keys(1 << 18, 4 + r, "u31") for r in range(p)]
    base = 0
    vs = []
    for k in ks:  # payload = the element's global index in the concatenation
        vs.append(np.arange(base, base + k.size, dtype=np.uint32))
        base += k.size
    return ks, vs


def _worker(rank, p, port, outdir):
    res = {"rank": rank, "ok": True, "errors": []}
    try:
        import torch.distributed as dist

        import oracle
        import paper_2211_16479_b200 as ms

        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=p, device_id=dev)
        comm = ms.Comm()

        def fail(msg):
            res["ok"] = False
            res["errors"].append(msg)

        def check_balanced(comm_, tag):
            for case in ("unequal", "equal", "int64"):
                ks, vs = _shards(p, case)
                cat = np.concatenate(ks)
                catv = np.concatenate(vs)
                ek, ev = oracle.sort(cat, catv)
                esplit = oracle.split_matrix(ks)
                K = np.concatenate([[0], np.cumsum([k.size for k in ks])])
                for pairs in (False, True):
                    for mode in (0, 1):
                        ms.set_exchange_mode(mode)
                        kd = torch.from_numpy(ks[rank].copy()).to(dev)
                        vd = (torch.from_numpy(vs[rank].view(np.int32).copy()).to(dev)
                              if pairs else None)
                        _, _, split = ms.msort_sort_distributed(kd, comm_, vals=vd,
                                                                return_split=True)
                        torch.cuda.synchronize()
                        a, b = int(K[rank]), int(K[rank + 1])
                        name = f"{tag}/{case}/pairs={pairs}/mode={mode}"
                        if not np.array_equal(split, esplit):
                            fail(f"{name}: split matrix differs")
                        if not np.array_equal(kd.cpu().numpy(), ek[a:b]):
                            fail(f"{name}: keys differ from the oracle slice")
                        if pairs and not np.array_equal(vd.cpu().numpy().view(np.uint32), ev[a:b]):
                            fail(f"{name}: payload differs from the oracle slice")
                ms.set_exchange_mode(0)

        check_balanced(comm, "own-comm")
        # the reserved pull exchange: no host synchronisation inside the call
        # (keys, 3..8 ranks); output checked after a device sync
        if p >= 3:
            ks, _ = _shards(p, "equal")
            cat = np.concatenate(ks)
            ek = oracle.sort(cat)
            comm.reserve(max(k.size for k in ks))
            comm.set_exchange(1)  # per communicator (msort_comm_set_exchange)
            for rep in range(3):
                kd = torch.from_numpy(ks[rank].copy()).to(dev)
                ms.msort_sort_distributed(kd, comm)
                torch.cuda.synchronize()
                a = rank * ks[0].size
                if not np.array_equal(kd.cpu().numpy(), ek[a:a + ks[rank].size]):
                    fail(f"reserved pull rep {rep}: keys differ from the oracle slice")
            comm.set_exchange(-1)
        # the paper's rank tree (f4): rank 0 gathers everything
        for pairs in (False, True):
            ks, vs = _shards(p, "unequal")
            kd = torch.from_numpy(ks[rank].copy()).to(dev)
            vd = torch.from_numpy(vs[rank].view(np.int32).copy()).to(dev) if pairs else None
            rk, rv = ms.msort_sort_distributed_tree(kd, comm, in_vals=vd)
            torch.cuda.synchronize()
            if rank == 0:
                exp = oracle.sort_tree(ks, vs if pairs else None)
                ek, ev = (exp if pairs else (exp, None))
                if not np.array_equal(rk.cpu().numpy(), ek):
                    fail(f"tree/pairs={pairs}: keys differ from oracle.sort_tree")
                if pairs and not np.array_equal(rv.cpu().numpy().view(np.uint32), ev):
                    fail(f"tree/pairs={pairs}: payload differs from oracle.sort_tree")
        comm.close()
        # on torch's own NCCL communicator (non-owning wrap)
        wrapped = ms.Comm.from_torch(device=dev)
        check_balanced(wrapped, "torch-comm")
        wrapped.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001 -- reported to the parent
        res["ok"] = False
        res["errors"].append(traceback.format_exc()[-3000:])
    with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs (one NCCL rank per GPU)")
@pytest.mark.parametrize("p", sorted({2, min(NGPU, 4), min(NGPU, 8)} - {0, 1}))
def test_nccl_multi_gpu(p, tmp_path):
    import torch.multiprocessing as mp

    port = _free_port()
    mp.start_processes(_worker, args=(p, port, str(tmp_path)), nprocs=p, join=True,
                       start_method="spawn")
    errs = []
    for r in range(p):
        with open(tmp_path / f"rank{r}.json") as f:
            d = json.load(f)
        if not d["ok"]:
            errs.append(f"rank {r}: " + " | ".join(d["errors"]))
    assert not errs, "\n".join(errs)
