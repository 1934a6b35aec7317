"""ctypes wrapper of the CPU oracle (oracle/msort_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this module.  The product
path (paper_2211_16479_b200) never imports it and shares no code with it.

All functions take and return numpy arrays on the host; they copy their input
(the paper's sorts are pure functions) unless named `*_inplace`.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libmsort_oracle.so")

_KD = {np.dtype(np.int32): 0, np.dtype(np.uint32): 1, np.dtype(np.int64): 2, np.dtype(np.uint64): 3}


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no CUDA)."""
    src = os.path.join(_HERE, "msort_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "msort_oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-fPIC", "-shared", "-pthread",
             src, "-o", _SO + ".tmp"]
        )
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        vp, sz, u32p, i64p = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p
        L.msort_oracle_sort.argtypes = [vp, u32p, sz, ctypes.c_int]
        L.msort_oracle_merge.argtypes = [vp, u32p, sz, vp, u32p, sz, vp, u32p, ctypes.c_int]
        L.msort_oracle_split_matrix.argtypes = [ctypes.POINTER(ctypes.c_void_p),
                                                ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                                ctypes.c_int, i64p]
        L.msort_oracle_check.argtypes = [vp, vp, u32p, sz, ctypes.c_int]
        L.msort_oracle_paper_mp.argtypes = [vp, u32p, sz, ctypes.c_int, ctypes.c_int]
        for f in ("msort_oracle_sort", "msort_oracle_merge", "msort_oracle_split_matrix",
                  "msort_oracle_check", "msort_oracle_paper_mp"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _kd(a: np.ndarray) -> int:
    try:
        return _KD[a.dtype]
    except KeyError:
        raise TypeError(f"oracle: unsupported key dtype {a.dtype}") from None


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _rc(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"{what} failed with {rc}")


def sort_inplace(keys: np.ndarray, vals: np.ndarray | None = None) -> None:
    assert keys.flags.c_contiguous and keys.ndim == 1
    if vals is not None:
        assert vals.dtype == np.uint32 and vals.shape == keys.shape and vals.flags.c_contiguous
    _rc(lib().msort_oracle_sort(_ptr(keys), _ptr(vals), keys.size, _kd(keys)), "oracle sort")


def sort(keys: np.ndarray, vals: np.ndarray | None = None):
    """Stable ascending sort.  Returns keys, or (keys, vals)."""
    k = np.ascontiguousarray(keys).copy()
    v = None if vals is None else np.ascontiguousarray(vals, dtype=np.uint32).copy()
    sort_inplace(k, v)
    return k if vals is None else (k, v)


def sort_segmented(keys: np.ndarray, offsets, vals: np.ndarray | None = None):
    """Batched sort (include/msort.h msort_sort_segmented): the stable sort of
    P:77-84 applied to every segment keys[off[i]:off[i+1]] on its own.
    Returns keys, or (keys, vals)."""
    k = np.ascontiguousarray(keys).copy()
    v = None if vals is None else np.ascontiguousarray(vals, dtype=np.uint32).copy()
    off = np.asarray(offsets, dtype=np.int64)
    for i in range(off.size - 1):
        a, b = int(off[i]), int(off[i + 1])
        if b - a >= 2:
            ks = k[a:b].copy()
            vs = None if v is None else v[a:b].copy()
            sort_inplace(ks, vs)
            k[a:b] = ks
            if v is not None:
                v[a:b] = vs
    return k if vals is None else (k, v)


def merge(a, b, av=None, bv=None):
    """merge(left, right), ties to the left run (reading R1)."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b, dtype=a.dtype)
    out = np.empty(a.size + b.size, dtype=a.dtype)
    withv = av is not None
    outv = np.empty(out.size, dtype=np.uint32) if withv else None
    if withv:
        av = np.ascontiguousarray(av, dtype=np.uint32)
        bv = np.ascontiguousarray(bv, dtype=np.uint32)
    _rc(lib().msort_oracle_merge(_ptr(a), _ptr(av), a.size, _ptr(b), _ptr(bv), b.size,
                                 _ptr(out), _ptr(outv), _kd(a)), "oracle merge")
    return out if not withv else (out, outv)


def sort_tree(shards, vals=None):
    """The paper's MPI merge (fig. mpi-merge-code) run literally on
    host arrays: every rank's array sorted (the subsort), then
        split = size / 2
        while split >= 1:
            ranks in [split, 2 split) send `local` to rank - split;
            ranks < split: local = merge(local, received)
            split = split / 2
    Rank 0's final array is returned (keys, or (keys, vals)).  For world sizes
    that are not powers of two the halving keeps ceil(active / 2) parents with
    the same pairing rank <- rank + split (reading R13)."""
    local = [sort(np.asarray(k)) if vals is None else sort(np.asarray(k), np.asarray(v))
             for k, v in zip(shards, vals if vals is not None else [None] * len(shards))]
    active = len(local)
    while active > 1:
        split = (active + 1) // 2  # = size / 2 when active is a power of two
        for rank in range(active - split):
            child = rank + split
            if vals is None:
                local[rank] = merge(local[rank], local[child])
            else:
                local[rank] = merge(local[rank][0], local[child][0], local[rank][1],
                                    local[child][1])
        active = split
    return local[0]


def tree_rank_order(p: int) -> list:
    """The order in which sort_tree's merges leave the ranks' elements among
    equal keys: rank 0's parent-first merges concatenate subtrees."""
    order = [[r] for r in range(p)]
    active = p
    while active > 1:
        split = (active + 1) // 2
        for rank in range(active - split):
            order[rank] = order[rank] + order[rank + split]
        active = split
    return order[0]


def split_matrix(shards) -> np.ndarray:
    """(p+1) x p reference split matrix of the distributed sort (reading R10/R11)."""
    p = len(shards)
    shards = [np.ascontiguousarray(s) for s in shards]
    dt = shards[0].dtype
    assert all(s.dtype == dt for s in shards)
    ptrs = (ctypes.c_void_p * p)(*[s.ctypes.data for s in shards])
    sizes = (ctypes.c_size_t * p)(*[s.size for s in shards])
    out = np.zeros((p + 1, p), dtype=np.int64)
    _rc(lib().msort_oracle_split_matrix(ptrs, sizes, p, _KD[dt], _ptr(out)), "oracle split")
    return out


def check(in_keys, out_keys, out_vals=None) -> int:
    """Invariant bit mask: 1 unsorted, 2 not a permutation, 4 unstable."""
    in_keys = np.ascontiguousarray(in_keys)
    out_keys = np.ascontiguousarray(out_keys, dtype=in_keys.dtype)
    if out_vals is not None:
        out_vals = np.ascontiguousarray(out_vals, dtype=np.uint32)
    rc = lib().msort_oracle_check(_ptr(in_keys), _ptr(out_keys), _ptr(out_vals), in_keys.size,
                                  _kd(in_keys))
    if rc < 0:
        raise RuntimeError(f"oracle check failed with {rc}")
    return rc


def paper_mp_inplace(keys: np.ndarray, vals: np.ndarray | None = None, cores: int = 1) -> None:
    """The paper's multiprocessing merge sort on host threads."""
    _rc(lib().msort_oracle_paper_mp(_ptr(keys), _ptr(vals), keys.size, _kd(keys), int(cores)),
        "oracle paper_mp")
