"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Every expected value comes from oracle/ on the same seeded input.  Sizes span
several tiles and ragged tails; the BASELINE.json configs C1-C4 run at full
size, C5's per-GPU shard (2^28 int32, the bench workload) too.
"""
import os

import numpy as np
import pytest
import torch

import msort_inputs as mi

pytestmark = pytest.mark.gpu

NP_OF = {"i32": np.int32, "u32": np.uint32, "i64": np.int64, "u64": np.uint64}


@pytest.fixture(scope="module")
def ms():
    import paper_2211_16479_b200 as m

    assert torch.cuda.is_available()
    return m


def to_dev(a: np.ndarray) -> torch.Tensor:
    if a.dtype == np.uint32:
        return torch.from_numpy(a.view(np.int32)).cuda().view(torch.uint32)
    if a.dtype == np.uint64:
        return torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    return torch.from_numpy(a).cuda()


def to_host(t: torch.Tensor, dtype) -> np.ndarray:
    if t.dtype == torch.uint32:
        t = t.view(torch.int32)
    elif t.dtype == torch.uint64:
        t = t.view(torch.int64)
    return t.cpu().numpy().view(dtype)


def gpu_sort(ms, k: np.ndarray, v: np.ndarray | None):
    kd = to_dev(k)
    vd = to_dev(v) if v is not None else None
    ms.msort_sort_pairs(kd, vd)
    torch.cuda.synchronize()
    ok = to_host(kd, k.dtype)
    ov = to_host(vd, np.uint32) if v is not None else None
    return ok, ov


def oracle_sort(orc, k, v):
    if k.size >= (1 << 24):
        kk = k.copy()
        vv = None if v is None else v.copy()
        orc.paper_mp_inplace(kk, vv, os.cpu_count() or 1)
        return kk, vv
    if v is None:
        return orc.sort(k), None
    return orc.sort(k, v)


def check_parity(ms, orc, k, v):
    ok, ov = gpu_sort(ms, k, v)
    ek, ev = oracle_sort(orc, k, v)
    assert np.array_equal(ok, ek), f"keys differ at {np.nonzero(ok != ek)[0][:5]}"
    if v is not None:
        assert np.array_equal(ov, ev), f"payload differs at {np.nonzero(ov != ev)[0][:5]}"


def _keys(n, seed, dist, dtype):
    if dist == "dup":
        return mi.keys(n, seed, ("mod", 3)).astype(dtype)
    if dist == "eq":
        return np.full(n, 5, dtype=dtype)
    if dist == "asc":
        return np.arange(n).astype(dtype)
    if dist == "desc":
        return np.arange(n)[::-1].astype(dtype).copy()
    if dist == "ext":  # extremes of the dtype mixed with small values
        info = np.iinfo(dtype)
        pool = np.array([info.min, info.min + 1, 0, 1, info.max - 1, info.max], dtype=dtype)
        return pool[(mi.splitmix64(n, seed) % np.uint64(6)).astype(np.int64)]
    return mi.keys(n, seed, {np.int32: "i32", np.uint32: "u32", np.int64: "i64",
                             np.uint64: "u64"}[dtype])


@pytest.mark.parametrize("dtype", [np.int32, np.uint32, np.int64, np.uint64])
@pytest.mark.parametrize("pairs", [False, True])
def test_sizes_around_tiles(ms, orc, dtype, pairs):
    kd = {np.int32: 0, np.uint32: 1, np.int64: 2, np.uint64: 3}[dtype]
    T = ms.tile_size(kd, ms.MSORT_UINT32 if pairs else ms.MSORT_NONE)
    sizes = [0, 1, 2, 3, 17, T - 1, T, T + 1, 2 * T - 1, 2 * T, 2 * T + 1, 3 * T + 5, 5 * T - 3,
             8 * T, 8 * T + 1, (1 << 17) - 1, (1 << 17) + 1, 123457]
    for i, n in enumerate(sizes):
        for dist in ("rand", "dup"):
            k = _keys(n, 100 + i, dist, dtype)
            v = mi.index_payload(n) if pairs else None
            check_parity(ms, orc, k, v)


@pytest.mark.parametrize("dist", ["eq", "asc", "desc", "ext", "dup"])
@pytest.mark.parametrize("dtype", [np.int32, np.uint32, np.int64, np.uint64])
def test_structured_inputs(ms, orc, dist, dtype):
    for n in (4096 * 5 + 77, 300001):
        check_parity(ms, orc, _keys(n, 7, dist, dtype), mi.index_payload(n))
        check_parity(ms, orc, _keys(n, 8, dist, dtype), None)


def test_misaligned_views(ms, orc):
    """Pointers aligned to the element but not to 16 bytes (offsets 1-3)."""
    n = 50000
    for off in (1, 2, 3):
        base = mi.keys(n + off, 11 + off, "i32")
        vals = mi.index_payload(n + off)
        kd = to_dev(base)[off:]
        vd = to_dev(vals)[off:]
        ms.msort_sort_pairs(kd, vd)
        torch.cuda.synchronize()
        ek, ev = orc.sort(base[off:].copy(), vals[off:].copy())
        assert np.array_equal(to_host(kd, np.int32), ek)
        assert np.array_equal(to_host(vd, np.uint32), ev)


def test_invalid_arguments(ms):
    import ctypes

    L = ms.lib
    assert L.msort_sort(None, 0, 0, None) == 0  # n == 0: no-op
    t = torch.zeros(8, dtype=torch.int32, device="cuda")
    assert L.msort_sort(ctypes.c_void_p(t.data_ptr() + 2), 4, 0, None) == 1  # misaligned
    assert L.msort_sort(ctypes.c_void_p(t.data_ptr()), 4, 7, None) == 1  # bad dtype
    assert L.msort_sort_pairs(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(t.data_ptr() + 8), 4,
                              0, 1, None) == 1  # overlap
    assert L.msort_sort_pairs(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(t.data_ptr() + 16), 2,
                              0, 2, None) == 2  # 8-byte payload not built


def test_convenience_calls_allocate(ms, orc):
    """msort_sort / msort_sort_pairs (library-allocated workspace)."""
    import ctypes

    n = 70001
    k = mi.keys(n, 3, "u32")
    kd = to_dev(k)
    st = ms.lib.msort_sort(ctypes.c_void_p(kd.data_ptr()), n, ms.MSORT_UINT32,
                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0
    torch.cuda.synchronize()
    assert np.array_equal(to_host(kd, np.uint32), orc.sort(k))


# ----------------------------------------------------- BASELINE.json configs
def test_c1(ms, orc):
    k, _ = mi.config_input("C1")
    check_parity(ms, orc, k, None)


def test_c2_random_sorted_reversed(ms, orc):
    k, _ = mi.config_input("C2")
    ek = oracle_sort(orc, k, None)[0]
    for variant in (k, ek, ek[::-1].copy()):  # reading R8: C2s / C2r
        ok, _ = gpu_sort(ms, variant, None)
        assert np.array_equal(ok, ek)


def test_c3_int64_duplicates_stability(ms, orc):
    k, v = mi.config_input("C3")
    ok, ov = gpu_sort(ms, k, v)
    assert orc.check(k, ok, ov) == 0
    ek, ev = oracle_sort(orc, k, v)
    assert np.array_equal(ok, ek) and np.array_equal(ov, ev)
    # SURVEY.md §8(c) stability pin: first three key-0 payloads
    assert ov[:3].tolist() == [108, 739, 1575]


def test_c4_uint32_pairs(ms, orc):
    k, v = mi.config_input("C4")
    ok, ov = gpu_sort(ms, k, v)
    ek, ev = oracle_sort(orc, k, v)
    assert np.array_equal(ok, ek) and np.array_equal(ov, ev)


def test_c5_shard_full_size(ms, orc):
    """The bench workload: one 2^28 int32 shard (seed 4), bit-exact."""
    n = 1 << 28
    kd = mi.keys_torch(n, 4, "u31", device="cuda")
    k = kd.cpu().numpy()
    ms.msort_sort(kd)
    torch.cuda.synchronize()
    ek = k.copy()
    orc.paper_mp_inplace(ek, None, os.cpu_count() or 1)
    assert np.array_equal(kd.cpu().numpy(), ek)


def test_torch_generator_on_gpu_matches_numpy():
    for dist in ("u31", "u32", ("mod", 1000), "i64"):
        a = mi.keys(1 << 20, 9, dist)
        b = mi.keys_torch(1 << 20, 9, dist, device="cuda")
        assert np.array_equal(a, to_host(b, a.dtype))


@pytest.mark.parametrize("pinned", [True, False])
def test_sort_host_entry_point(ms, orc, pinned):
    """msort_sort_host: host -> device -> sort -> host, keys and pairs."""
    n = 300007
    k = mi.keys(n, 12, "i64")
    v = mi.index_payload(n)
    hk = torch.from_numpy(k.copy())
    hv = torch.from_numpy(v.view(np.int32).copy())
    if pinned:
        hk, hv = hk.pin_memory(), hv.pin_memory()
    ok = torch.empty_like(hk)
    ov = torch.empty_like(hv)
    if pinned:
        ok, ov = ok.pin_memory(), ov.pin_memory()
    dk = torch.empty(n, dtype=torch.int64, device="cuda")
    dv = torch.empty(n, dtype=torch.int32, device="cuda")
    ms.msort_sort_host(hk, ok, dk, host_vals=hv, host_vals_out=ov, dev_vals=dv)
    torch.cuda.synchronize()
    ek, ev = orc.sort(k, v)
    assert np.array_equal(ok.numpy(), ek)
    assert np.array_equal(ov.numpy().view(np.uint32), ev)
    assert np.array_equal(hk.numpy(), k)  # input untouched
    # keys only, in place on the host buffer
    hk2 = torch.from_numpy(mi.keys(n, 13, "u32").view(np.int32).copy())
    dk2 = torch.empty(n, dtype=torch.int32, device="cuda").view(torch.uint32)
    ms.msort_sort_host(hk2.view(torch.uint32), hk2.view(torch.uint32), dk2)
    torch.cuda.synchronize()
    assert np.array_equal(hk2.numpy().view(np.uint32), orc.sort(mi.keys(n, 13, "u32")))


def test_random_sizes_stress(ms, orc):
    """60 random (size, dtype, distribution, payload) combinations, sizes up to
    2^21 + ragged tails: every one bit-exact to the oracle."""
    rng = np.random.default_rng(2211)
    dts = [np.int32, np.uint32, np.int64, np.uint64]
    dists = ["rand", "dup", "eq", "asc", "desc", "ext"]
    for t in range(60):
        n = int(rng.integers(0, 1 << int(rng.integers(1, 22))))
        dtype = dts[int(rng.integers(0, 4))]
        dist = dists[int(rng.integers(0, len(dists)))]
        pairs = bool(rng.integers(0, 2))
        k = _keys(n, 5000 + t, dist, dtype)
        v = mi.index_payload(n) if pairs else None
        check_parity(ms, orc, k, v)


# ---- K0: keys-only sorts of n <= 69632 in one cluster launch
K0_SIZES = [2, 3, 31, 100, 1000, 4097, 8191, 8192, 8193, 12000, 16384, 16385, 30001, 32768,
            32769, 50000, 65535, 65536, 65537, 69632]


@pytest.mark.parametrize("dtype", [np.int32, np.uint32, np.int64, np.uint64])
def test_small_cluster_sort_sizes(ms, orc, dtype):
    """Every cluster size (1, 2, 4, 8 CTAs), ragged chunks, the K0 / general
    path boundary (65536 / 65537), against the oracle."""
    for i, n in enumerate(K0_SIZES):
        for dist in ("rand", "dup"):
            check_parity(ms, orc, _keys(n, 900 + i, dist, dtype), None)


@pytest.mark.parametrize("dist", ["eq", "asc", "desc", "ext"])
def test_small_cluster_sort_structured(ms, orc, dist):
    for dtype in (np.int32, np.uint64):
        for n in (8704, 20000, 65536):
            check_parity(ms, orc, _keys(n, 7, dist, dtype), None)


@pytest.mark.parametrize("mode", ["2", "3", "4"])
def test_small_cluster_sort_variants(ms, orc, mode, monkeypatch):
    """Every K0 variant at every cluster size (MSORT_K0 is read per call):
    4 = the one-step multiway cluster merge also for 2-CTA clusters (the
    default uses it from 4 CTAs on), 3 = pairwise cluster levels, 2 = the
    same without the warp-shuffle network."""
    monkeypatch.setenv("MSORT_K0", mode)
    for i, n in enumerate([4097, 6000, 8192, 8193, 16384, 24577, 32768, 40000, 65535, 65536]):
        for dtype in (np.int32, np.uint64):
            for dist in ("rand", "dup", "eq", "desc"):
                check_parity(ms, orc, _keys(n, 300 + i, dist, dtype), None)


def test_small_cluster_sort_c1_out_of_place_and_graph(ms, orc):
    """C1 (2^16 int32, seed 0) out of place, then captured in a CUDA graph and
    replayed on new data: bit-exact every time."""
    k, _ = mi.config_input("C1")
    kin = to_dev(k)
    kout = torch.empty_like(kin)
    ws = ms.workspace(k.size, torch.int32, False, device="cuda")
    ms.msort_sort_out(kin, kout, ws=ws)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(kout, np.int32), orc.sort(k))
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            ms.msort_sort_out(kin, kout, ws=ws, stream=s)
    for seed in (11, 12):
        k2 = mi.keys(k.size, seed, "i32")
        kin.copy_(to_dev(k2))
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(to_host(kout, np.int32), orc.sort(k2))


# ---- K3 chunk scheduling: single-chunk grabs whose co-ranks are searched by
# lane groups (edges by 16 lanes, inner ones inside the edges' bracket), with
# ragged last chunks at every level and chunk sizes 1..8 tiles
@pytest.mark.parametrize("n,dist,dtype,pairs", [
    ((1 << 21) + 4321, "rand", np.int32, False),     # chunks of 1 tile
    (9 * (1 << 20) + 77, "dup", np.int32, False),    # 2-tile chunks, heavy ties
    ((1 << 24) + 12345, "rand", np.uint32, False),   # 3-tile chunks (C2 + a tail)
    (3 * (1 << 24) + 11, "rand", np.int32, False),   # 8-tile chunks, one per grab
    ((1 << 25) - 5, "dup", np.int64, True),          # 8-byte keys + payload
    ((1 << 26) + 999, "rand", np.int32, False),      # 2^26: single-chunk grabs
])
def test_k3_single_chunk_grabs(ms, orc, n, dist, dtype, pairs):
    k = _keys(n, 7100 + n % 97, dist, dtype)
    v = mi.index_payload(n) if pairs else None
    check_parity(ms, orc, k, v)


# ---- key-range narrowing: 8-byte keys spanning < 2^32 values sort as 32-bit
# offsets (Kernels::sort_narrowed); the choice is made on the device
def _range_keys(n, seed, dtype, lo, span):
    """n keys of `dtype` uniform in [lo, lo + span) (span <= 2^63), plus both ends."""
    rng = np.random.default_rng(seed)
    off = rng.integers(0, span, size=n, dtype=np.uint64)
    if np.dtype(dtype) == np.int64:
        k = (np.int64(lo) + off.astype(np.int64)).astype(np.int64)
    else:
        k = (np.uint64(lo) + off).astype(np.uint64)
    if n >= 2:
        k[n // 3] = np.asarray(lo).astype(dtype)
        k[(2 * n) // 3] = (np.asarray(lo).astype(dtype) + np.asarray(span - 1).astype(dtype))
    return k


@pytest.mark.parametrize("dtype", [np.int64, np.uint64])
@pytest.mark.parametrize("pairs", [False, True])
def test_key_range_narrowing(ms, orc, dtype, pairs):
    """Spans just below / at / above 2^32 (narrowed / narrowed / 8-byte path),
    negative and extreme bases, ragged sizes above the K0 limit."""
    big = (1 << 63) - (1 << 33) if dtype == np.int64 else (1 << 64) - (1 << 33)
    cases = [(0, 1000), (-(1 << 40) if dtype == np.int64 else 1 << 40, (1 << 32) - 1),
             (-(1 << 63) if dtype == np.int64 else 0, 1 << 32),
             (big, (1 << 32) + 1), (5, 1 << 40), (7, 1)]
    for i, (lo, span) in enumerate(cases):
        for n in (65537, 3 * 8704 + 5, (1 << 20) + 333):
            k = _range_keys(n, 40 + i, dtype, lo, span)
            v = mi.index_payload(n) if pairs else None
            check_parity(ms, orc, k, v)


def test_key_range_narrowing_out_of_place_and_off(ms, orc, monkeypatch):
    """Out of place with a workspace, C3-shaped keys; and the same with the
    narrowing disabled (MSORT_NARROW=0): identical to the oracle both ways."""
    n = (1 << 22) + 17
    k = mi.keys(n, 2, ("mod", 1000)).astype(np.int64)
    v = mi.index_payload(n)
    ek, ev = orc.sort(k, v)
    for mode in ("1", "0"):
        monkeypatch.setenv("MSORT_NARROW", mode)
        kin, vin = to_dev(k), to_dev(v)
        kout, vout = torch.empty_like(kin), torch.empty_like(vin)
        ws = ms.workspace(n, torch.int64, True, device="cuda")
        ms.msort_sort_out(kin, kout, in_vals=vin, vals_out=vout, ws=ws)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(kout, np.int64), ek)
        assert np.array_equal(to_host(vout, np.uint32), ev)
        assert np.array_equal(to_host(kin, np.int64), k)  # input untouched
