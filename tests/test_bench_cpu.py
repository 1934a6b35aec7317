"""bench.py's reference arm (the CPU oracle on a bounded sample) runs on CPU and
prints one JSON line with the contract's keys; the GPU arm's argument parser
accepts the driver's flags."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["value"] > 0 and d["unit"] == "keys/s" and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def test_parser_accepts_driver_flags():
    sys.path.insert(0, ROOT)
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    old = sys.argv
    try:
        sys.argv = ["bench.py", "--gpus", "8", "--steps", "10", "--warmup", "3", "--impl",
                    "native", "--exchange", "pull", "--no-e2e", "--no-batched"]
        a = mod.parse()
    finally:
        sys.argv = old
    assert (a.gpus, a.steps, a.warmup, a.exchange) == (8, 10, 3, "pull")


def _bench_module():
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod2", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


class _FakeDist:
    """torch.distributed stand-in for one rank: all_reduce(MIN) combines the
    local flag with the other ranks' (given) flags."""

    class ReduceOp:
        MIN = "min"

    def __init__(self, others):
        self.others = others

    def all_reduce(self, t, op=None):
        t.fill_(min([int(t.item())] + list(self.others)))


class _FakeMs:
    def __init__(self, fail_sort=False):
        self.mode = None
        self.fail_sort = fail_sort

    def set_exchange_mode(self, m):
        self.mode = m

    def msort_sort_distributed_out(self, kin, kout, comm, ws=None, stream=None, return_split=False):
        import torch

        if self.fail_sort:
            raise RuntimeError("simulated IPC failure")
        kout.copy_(torch.sort(kin)[0])
        return kout, None, [[0], [kin.numel()]]


class _FakeComm:
    def __init__(self, ms):
        self.ms = ms

    def set_exchange(self, m):
        self.ms.mode = m

    def reserve(self, n, keys_dtype=None, with_vals=False, stream=None):
        self.reserved = n


def _choose(monkeypatch, exchange, others, fail_sort=False):
    import argparse

    import torch

    mod = _bench_module()
    monkeypatch.setattr(torch.cuda, "synchronize", lambda *a, **k: None)
    ms = _FakeMs(fail_sort)
    kin = torch.randint(0, 1000, (4096,), dtype=torch.int32)
    kout = torch.empty_like(kin)
    args = argparse.Namespace(exchange=exchange)
    last = [None]
    got = mod.choose_exchange(args, ms, _FakeComm(ms), _FakeDist(others), "cpu", kin, kout, None,
                              None, 2, 0, kin.numel(), last)
    return got, ms.mode, last[0]


def test_choose_exchange_agreement(monkeypatch):
    """bench.py N > 1: the pull exchange is used only when the verified first
    step succeeds on EVERY rank (MIN over ranks); otherwise all ranks take
    the all-to-all together ("auto") or fail together ("pull")."""
    import pytest

    got, mode, split = _choose(monkeypatch, "auto", [1])
    assert got == "pull" and mode == 1 and split is not None
    got, mode, _ = _choose(monkeypatch, "auto", [0])  # another rank failed
    assert got.startswith("alltoall") and mode == 0
    got, mode, _ = _choose(monkeypatch, "auto", [1], fail_sort=True)  # this rank failed
    assert got.startswith("alltoall") and mode == 0 and "simulated" in got
    got, mode, _ = _choose(monkeypatch, "alltoall", [1])
    assert got == "alltoall" and mode == 0
    with pytest.raises(RuntimeError):
        _choose(monkeypatch, "pull", [0])
