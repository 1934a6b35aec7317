"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO sorting arithmetic: it only draws keys. It is the one
piece that both sides of the parity check use (the CUDA path never imports
`oracle/`, the oracle never imports the CUDA path).

Generator (SURVEY.md §8(c) reading L6): counter-mode
SplitMix64.  Output i for seed s is

    z_i = mix(s + (i + 1) * 0x9E3779B97F4A7C15  mod 2^64)
    mix(z): z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
            z = (z ^ (z >> 27)) * 0x94D049BB133111EB
            return z ^ (z >> 31)

which equals the i-th output of the sequential SplitMix64 seeded with s, so
it can be drawn in parallel and in chunks with bit-identical results.  The
paper draws `np.random.randint(n, size=n)` unseeded (Fig.
fig:mpi-scatter-code), so a named, seeded generator is our reading.

Mappings from z to a key (the `dist` argument):

    "u31"      int32 in [0, 2^31)       (int32)(z >> 33)      configs C1, C2, C5
    "u32"      uint32 full range        (uint32)(z >> 32)     config C4
    "i32"      int32 full signed range  bit pattern of z >> 32 (edge tests)
    "i64"      int64 full signed range  bit pattern of z      (edge tests)
    "u64"      uint64 full range        z                      (edge tests)
    ("mod", m) int64 in [0, m), m < 2^32: multiply-high (z * m) >> 64
                                                              config C3 (m = 1000)

Payloads for pairs are the original index i (uint32), SURVEY.md §8(c) L9.
"""
from __future__ import annotations

import numpy as np

GOLDEN_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

_CHUNK = 1 << 22


def _mix(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    return z ^ (z >> np.uint64(31))


def splitmix64(n: int, seed: int, start: int = 0) -> np.ndarray:
    """Raw 64-bit outputs z_start .. z_{start+n-1} for `seed` (uint64 array)."""
    with np.errstate(over="ignore"):
        idx = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        return _mix(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + idx * GOLDEN_GAMMA)


def _map(z: np.ndarray, dist) -> np.ndarray:
    if dist == "u31":
        return (z >> np.uint64(33)).astype(np.int32)
    if dist == "u32":
        return (z >> np.uint64(32)).astype(np.uint32)
    if dist == "i32":
        return (z >> np.uint64(32)).astype(np.uint32).view(np.int32)
    if dist == "i64":
        return z.view(np.int64)
    if dist == "u64":
        return z
    if isinstance(dist, tuple) and dist[0] == "mod":
        m = int(dist[1])
        assert 0 < m < (1 << 32)
        mm = np.uint64(m)
        hi = z >> np.uint64(32)
        lo = z & np.uint64(0xFFFFFFFF)
        # high 64 bits of the 128-bit product z*m, exact for m < 2^32
        return ((hi * mm + ((lo * mm) >> np.uint64(32))) >> np.uint64(32)).astype(np.int64)
    raise ValueError(f"unknown dist {dist!r}")


DTYPE_OF = {"u31": np.int32, "u32": np.uint32, "i32": np.int32, "i64": np.int64, "u64": np.uint64}


def keys(n: int, seed: int, dist="u31", out: np.ndarray | None = None) -> np.ndarray:
    """n seeded keys with mapping `dist`; generated in chunks to bound host memory."""
    dt = np.int64 if isinstance(dist, tuple) else DTYPE_OF[dist]
    if out is None:
        out = np.empty(n, dtype=dt)
    assert out.dtype == dt and out.shape == (n,)
    with np.errstate(over="ignore"):
        for s in range(0, n, _CHUNK):
            e = min(n, s + _CHUNK)
            out[s:e] = _map(splitmix64(e - s, seed, s), dist)
    return out


def _i64(c: int) -> int:
    """A 64-bit constant as the signed int64 with the same bits."""
    return c - (1 << 64) if c >= (1 << 63) else c


def _srl(z, s: int):
    """Logical right shift of int64 torch tensors (bit pattern of uint64)."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def keys_torch(n: int, seed: int, dist="u31", device="cuda", start: int = 0):
    """The same counter-mode SplitMix64 keys as `keys`, drawn with torch int64
    ops (wrap-around multiply, masked shifts) on any device -- bit-identical to
    the numpy version (tests/test_oracle.py::test_torch_generator_matches).
    Used to build large inputs on the GPU quickly; pure plumbing."""
    import torch

    idx = torch.arange(start + 1, start + n + 1, dtype=torch.int64, device=device)
    z = idx * _i64(int(GOLDEN_GAMMA)) + _i64(seed & 0xFFFFFFFFFFFFFFFF)
    z = (z ^ _srl(z, 30)) * _i64(int(_M1))
    z = (z ^ _srl(z, 27)) * _i64(int(_M2))
    z = z ^ _srl(z, 31)
    del idx
    if dist == "u31":
        return _srl(z, 33).to(torch.int32)
    if dist in ("u32", "i32"):
        hi = _srl(z, 32)
        hi = torch.where(hi >= (1 << 31), hi - (1 << 32), hi).to(torch.int32)
        return hi.view(torch.uint32) if dist == "u32" else hi
    if dist == "i64":
        return z
    if dist == "u64":
        return z.view(torch.uint64)
    if isinstance(dist, tuple) and dist[0] == "mod":
        m = int(dist[1])
        assert 0 < m < (1 << 31)
        hi = _srl(z, 32)
        lo = z & 0xFFFFFFFF
        return _srl(hi * m + _srl(lo * m, 32), 32)
    raise ValueError(f"unknown dist {dist!r}")


def index_payload(n: int) -> np.ndarray:
    """Original-index payload v_i = i (uint32), used to observe stability."""
    assert n <= (1 << 32)
    return np.arange(n, dtype=np.uint32)


# The BASELINE.json configs (SURVEY.md §0 table, §8(c) mappings).
CONFIGS = {
    "C1": dict(n=1 << 16, seed=0, dist="u31", pairs=False),
    "C2": dict(n=1 << 24, seed=1, dist="u31", pairs=False),
    "C3": dict(n=1 << 26, seed=2, dist=("mod", 1000), pairs=True),
    "C4": dict(n=1 << 27, seed=3, dist="u32", pairs=True),
    "C5": dict(n=1 << 28, seed=4, dist="u31", pairs=False),  # seed 4 + rank
}


def config_input(name: str, rank: int = 0, n: int | None = None):
    """(keys, vals-or-None) for a BASELINE.json config; C5 uses seed 4 + rank."""
    c = CONFIGS[name]
    nn = c["n"] if n is None else n
    seed = c["seed"] + (rank if name == "C5" else 0)
    k = keys(nn, seed, c["dist"])
    v = index_payload(nn) if c["pairs"] else None
    return k, v
