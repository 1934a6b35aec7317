"""Pins of the CPU oracle against things other than itself (no GPU needed).

Each test names what fixes the expected value: brute force over all
permutations, the counting-rank definition, closed forms, numpy's stable sort
(a library routine), or the independent golden values of SURVEY.md §8(c).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import msort_inputs as mi

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

KEY_DTYPES = [np.int32, np.uint32, np.int64, np.uint64]


def _alphabet(dtype, m):
    """m distinct keys of `dtype` spanning the sign bit, so that a signed/
    unsigned mix-up or a wrong comparison changes the order."""
    dt = np.dtype(dtype)
    if dt.kind == "i":
        base = [np.iinfo(dt).min, -7, -1, 0, 1, 5, np.iinfo(dt).max]
    else:
        base = [0, 1, 5, (1 << (8 * dt.itemsize - 1)), (1 << (8 * dt.itemsize - 1)) + 3,
                np.iinfo(dt).max - 1, np.iinfo(dt).max]
    idx = np.linspace(0, len(base) - 1, m).round().astype(int) if m > 1 else [3]
    return np.array([base[i] for i in idx], dtype=dt)


def _brute_force_stable(keys):
    """All n! index permutations; keep those whose (key, index) sequence is
    strictly increasing lexicographically.  Returns the list of survivors."""
    n = len(keys)
    if n < 2:
        return [np.arange(n)]
    perms = np.array(list(itertools.permutations(range(n))), dtype=np.int64)
    k = keys[perms]
    ok = (k[:, :-1] < k[:, 1:]) | ((k[:, :-1] == k[:, 1:]) & (perms[:, :-1] < perms[:, 1:]))
    return perms[ok.all(axis=1)]


@pytest.mark.parametrize("dtype", KEY_DTYPES)
def test_brute_force_all_words(orc, dtype):
    """Every word over an m-letter alphabet, n <= 6: exactly one permutation
    satisfies the stable order, and the oracle (keys + index payload) is it."""
    for n in range(0, 7):
        for m in sorted({1, 2, 3, max(n, 1)}):
            if m ** n > 800 and n == 6 and m > 3:
                continue
            alpha = _alphabet(dtype, m)
            for word in itertools.product(range(m), repeat=n):
                keys = alpha[list(word)] if n else np.zeros(0, dtype=dtype)
                keys = np.asarray(keys, dtype=dtype)
                sols = _brute_force_stable(keys)
                assert len(sols) == 1
                ok, ov = orc.sort(keys, mi.index_payload(n))
                assert ov.tolist() == list(sols[0])
                assert ok.tolist() == keys[sols[0]].tolist()


def test_brute_force_all_permutations(orc):
    """Every permutation of 0..n-1 for n <= 7 sorts to the identity keys and
    the inverse permutation as payload (closed form for distinct keys)."""
    for n in range(0, 8):
        for perm in itertools.permutations(range(n)):
            keys = np.array(perm, dtype=np.int32)
            ok, ov = orc.sort(keys, mi.index_payload(n))
            assert ok.tolist() == list(range(n))
            inv = np.argsort(np.array(perm, dtype=np.int64)) if n else np.zeros(0, np.int64)
            assert ov.tolist() == inv.tolist()


@pytest.mark.parametrize("dtype", KEY_DTYPES)
@pytest.mark.parametrize("n,m", [(1000, 3), (2500, 40), (4096, 1 << 30), (3001, 1)])
def test_counting_rank_definition(orc, dtype, n, m):
    """pos(i) = #{j: k_j < k_i} + #{j < i: k_j = k_i},
    evaluated directly in O(n^2)."""
    z = mi.splitmix64(n, 1234 + n)
    alpha = _alphabet(dtype, 7)
    if m <= 7:
        keys = alpha[(z % np.uint64(m)).astype(np.int64)]
    else:
        keys = mi.keys(n, 99, {np.int32: "i32", np.uint32: "u32", np.int64: "i64",
                               np.uint64: "u64"}[dtype])
    keys = keys.astype(dtype)
    less = (keys[None, :] < keys[:, None]).sum(axis=1)
    eq_before = np.tril(keys[None, :] == keys[:, None], k=-1).sum(axis=1)
    pos = less + eq_before
    ok, ov = orc.sort(keys, mi.index_payload(n))
    assert np.array_equal(ok[pos], keys)
    assert np.array_equal(ov[pos], np.arange(n, dtype=np.uint32))


@pytest.mark.parametrize("dtype", KEY_DTYPES)
def test_library_stable_sort_cross_check(orc, dtype):
    """numpy's stable argsort (a library routine) at 2^18 with duplicates."""
    n = 1 << 18
    dist = {np.int32: "i32", np.uint32: "u32", np.int64: "i64", np.uint64: "u64"}[dtype]
    keys = mi.keys(n, 7, dist)
    keys = (keys >> 12) if dtype in (np.uint32, np.uint64) else (keys // 4096)  # duplicates
    keys = keys.astype(dtype)
    ok, ov = orc.sort(keys, mi.index_payload(n))
    ref = np.argsort(keys, kind="stable")
    assert np.array_equal(ov, ref.astype(np.uint32))
    assert np.array_equal(ok, keys[ref])


def test_closed_forms(orc):
    n = 10007
    asc = np.arange(n, dtype=np.int64) * 3 - 5000
    ok, ov = orc.sort(asc, mi.index_payload(n))
    assert np.array_equal(ok, asc) and np.array_equal(ov, np.arange(n))  # sorted -> identity
    rev = asc[::-1].copy()
    ok, ov = orc.sort(rev, mi.index_payload(n))
    assert np.array_equal(ok, asc) and np.array_equal(ov, np.arange(n)[::-1])  # reversal
    eq = np.full(n, 42, dtype=np.uint32)
    ok, ov = orc.sort(eq, mi.index_payload(n))
    assert np.array_equal(ov, np.arange(n))  # all equal -> identity payload (stability)
    for m in (0, 1):  # fewer than two elements: return
        k = np.array([7][:m], dtype=np.int32)
        assert orc.sort(k).tolist() == k.tolist()


def test_spec_examples(orc):
    """SPEC examples and the worked example of the
    first 16 C3 elements."""
    assert orc.merge(np.array([1, 3], np.int64), np.array([2, 4], np.int64)).tolist() == [1, 2, 3, 4]
    assert orc.merge(np.array([], np.int64), np.array([5], np.int64)).tolist() == [5]
    assert orc.sort(np.array([3, 1, 2], np.int64)).tolist() == [1, 2, 3]
    assert orc.sort(np.arange(10, dtype=np.int64)[::-1].copy()).tolist() == list(range(10))
    k = mi.keys(16, 2, ("mod", 1000))
    sk, sv = orc.sort(k, mi.index_payload(16))
    expect = [(203, 15), (250, 8), (311, 4), (339, 10), (346, 5), (373, 13), (437, 11), (555, 12),
              (591, 0), (595, 2), (726, 6), (727, 9), (739, 7), (749, 1), (765, 3), (932, 14)]
    assert list(zip(sk.tolist(), sv.tolist())) == expect


def test_merge_tie_rule_and_corank(orc):
    """merge() takes the left element on ties (reading R1); the co-rank
    i(d) = #A among the first d outputs satisfies the merge-path bounds."""
    rng = np.random.default_rng(5)
    for _ in range(400):
        na, nb = rng.integers(0, 12, size=2)
        a = np.sort(rng.integers(0, 4, size=na)).astype(np.int32)
        b = np.sort(rng.integers(0, 4, size=nb)).astype(np.int32)
        av = np.arange(na, dtype=np.uint32)
        bv = np.arange(na, na + nb, dtype=np.uint32)
        out, ov = orc.merge(a, b, av, bv)
        # the merge equals a stable sort of the concatenation (library routine)
        cat = np.concatenate([a, b])
        ref = np.argsort(cat, kind="stable")
        assert np.array_equal(ov, ref.astype(np.uint32)) and np.array_equal(out, cat[ref])
        for d in range(na + nb + 1):
            i = int(np.count_nonzero(ov[:d] < na))
            j = d - i
            assert 0 <= i <= na and 0 <= j <= nb
            if i > 0 and j < nb:
                assert a[i - 1] <= b[j]
            if j > 0 and i < na:
                assert b[j - 1] < a[i]


def test_check_detects_broken_outputs(orc):
    n = 1000
    keys = mi.keys(n, 3, ("mod", 50))
    ok, ov = orc.sort(keys, mi.index_payload(n))
    assert orc.check(keys, ok, ov) == 0
    bad = ok.copy(); bad[[10, 900]] = bad[[900, 10]]
    assert orc.check(keys, bad, ov) & 1
    badv = ov.copy(); badv[5] = badv[6]
    assert orc.check(keys, ok, badv) & 2
    # swap the payloads of two equal keys: still a permutation, but unstable
    t = int(np.nonzero(ok[1:] == ok[:-1])[0][0])
    uv = ov.copy(); uv[[t, t + 1]] = uv[[t + 1, t]]
    assert orc.check(keys, ok, uv) == 4


def _split_brute(shards):
    """Split matrix from Python's sorted() over (key, rank, index) tuples."""
    p = len(shards)
    recs = sorted((int(k), r, i) for r, s in enumerate(shards) for i, k in enumerate(s))
    K = np.concatenate([[0], np.cumsum([len(s) for s in shards])])
    out = np.zeros((p + 1, p), dtype=np.int64)
    for r in range(p + 1):
        for (_, j, _) in recs[: K[r]]:
            out[r, j] += 1
    return out


def test_split_matrix_definition(orc):
    rng = np.random.default_rng(11)
    for trial in range(300):
        p = int(rng.integers(1, 7))
        sizes = rng.integers(0, 9, size=p)
        if trial % 7 == 0:
            sizes[rng.integers(0, p)] = 0
        hi = int(rng.integers(1, 5))
        shards = [np.sort(rng.integers(-hi, hi, size=s)).astype(np.int64) for s in sizes]
        s = orc.split_matrix(shards)
        assert np.array_equal(s, _split_brute(shards))
        K = np.concatenate([[0], np.cumsum(sizes)])
        assert np.array_equal(s.sum(axis=1), K)
        assert (np.diff(s, axis=0) >= 0).all()
        assert np.array_equal(s[-1], sizes)


def test_paper_mp_equals_oracle(orc):
    for n, c in [(0, 3), (1, 4), (17, 4), (1000, 3), (100003, 8), (65536, 5)]:
        keys = mi.keys(n, 21, ("mod", 97))
        ok, ov = orc.sort(keys, mi.index_payload(n))
        k2, v2 = keys.copy(), mi.index_payload(n)
        orc.paper_mp_inplace(k2, v2, c)
        assert np.array_equal(k2, ok) and np.array_equal(v2, ov)


def test_generator_golden():
    """SplitMix64 seed 0 outputs (the widely published sequence) and the
    config first keys of SURVEY.md §8(c)."""
    z = mi.splitmix64(4, 0)
    assert [int(x) for x in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F,
                                   0xF88BB8A8724C81EC]
    assert mi.keys(8, 0, "u31").tolist() == [1896895516, 926699317, 56766092, 2084953172,
                                              228377781, 702926726, 373378399, 1656883613]
    assert mi.keys(8, 3, "u32").tolist() == [487265508, 3007737738, 2632706214, 312960251,
                                              929598893, 2732554039, 580447042, 3817016609]
    c5 = {0: [926544313, 1916429109, 1844940030, 1056077190],
          7: [679129662, 563424873, 1370185496, 1083650380]}
    for r, v in c5.items():
        assert mi.keys(4, 4 + r, "u31").tolist() == v
    # counter mode == chunked generation
    a = mi.splitmix64(1000, 9)
    b = np.concatenate([mi.splitmix64(300, 9, 0), mi.splitmix64(700, 9, 300)])
    assert np.array_equal(a, b)
    # multiply-high mapping stays in range and equals exact big-int arithmetic
    z = mi.splitmix64(200, 2)
    mh = mi.keys(200, 2, ("mod", 1000))
    assert mh.tolist() == [(int(x) * 1000) >> 64 for x in z]


# Independent numpy-derived values printed in SURVEY.md §8(c) "Golden values".
SURVEY = {
    "C1": dict(sum=70263081217147, duplicates=1,
               sorted_at=[19992, 535272919, 1071934641, 1607065802, 2147429601]),
    "C2": dict(sum=18015548003167332, duplicates=65329,
               sorted_at=[54, 537137808, 1073809295, 1610512162, 2147483627]),
    "C3": dict(sum=33516323853, sorted_at=[0, 0, 0, 499, 999],
               payload_at=[108, 739, 1575, 60858343, 67108710]),
    "C4": dict(sum=288217747904330091, duplicates=2075499,
               sorted_at=[66, 87, 90, 2147429140, 4294967157],
               payload_at=[98205384, 71266400, 41769820, 3259641, 106860143]),
}


def test_golden_file_matches_survey():
    """The oracle's full-size outputs (stored by make_golden.py, which calls
    only oracle/) agree with the survey's independent numpy computation."""
    with open(os.path.join(GOLDEN, "oracle_golden.json")) as f:
        g = json.load(f)
    for name, exp in SURVEY.items():
        got = g[name]
        assert got["sum"] == exp["sum"], name
        assert list(got["sorted_at"].values()) == exp["sorted_at"], name
        if "duplicates" in exp:
            assert got["duplicates"] == exp["duplicates"], name
        if "payload_at" in exp:
            assert list(got["payload_at"].values()) == exp["payload_at"], name
            assert got["check"] == 0


# SURVEY.md §8(c) addendum (independent numpy computation: np.sort per shard,
# value bisection, cross-checked by np.partition on the concatenation): the
# key at global position K_r = r * 2^28 of the C5 concatenation at p ranks,
# and every shard's min / max.
SURVEY_C5_VSTAR = {2: [1073704941], 4: [536879718, 1073750287, 1610621812],
                   8: [268433051, 536898611, 805317802, 1073767078, 1342188887, 1610616419,
                       1879055353]}
SURVEY_C5_MINMAX = [(14, 2147483646), (4, 2147483647), (18, 2147483633), (0, 2147483629),
                    (23, 2147483647), (1, 2147483635), (8, 2147483632), (5, 2147483640)]


def test_c5_digests_match_survey():
    """tests/golden/c5_digests.json (make_c5_digests.py: oracle only) against
    the survey's independent numbers: rank r's slice at p ranks starts with
    v*_r (its first key IS the key at K_r), the p = 1 slice spans shard 0's
    min..max, the p-rank slices span the min..max of the first p shards, and
    consecutive slices are ordered.  The slices' sums add up to the shards'
    sums (the generator, independent of the oracle)."""
    with open(os.path.join(GOLDEN, "c5_digests.json")) as f:
        g = json.load(f)
    assert g["n_per_rank"] == 1 << 28
    d = g["digests"]
    assert d["1"][0]["first"] == SURVEY_C5_MINMAX[0][0]
    assert d["1"][0]["last"] == SURVEY_C5_MINMAX[0][1]
    for p, vstar in SURVEY_C5_VSTAR.items():
        rows = d[str(p)]
        assert len(rows) == p
        assert [r["first"] for r in rows[1:]] == vstar, p
        assert rows[0]["first"] == min(m for m, _ in SURVEY_C5_MINMAX[:p])
        assert rows[-1]["last"] == max(m for _, m in SURVEY_C5_MINMAX[:p])
        assert all(rows[r]["last"] <= rows[r + 1]["first"] for r in range(p - 1))
        assert all(len(r["sha256"]) == 64 for r in rows)


def test_c5_digest_sums_match_generator():
    """The p = 1 and p = 2 digest rows sum to the generated shards' sums (the
    seeded generator alone, no sort): the slices are a permutation's worth of
    keys.  (p = 4, 8 would take a minute of numpy; their first keys are pinned
    above.)"""
    with open(os.path.join(GOLDEN, "c5_digests.json")) as f:
        d = json.load(f)["digests"]
    n = 1 << 28
    sums = []
    for r in range(2):
        t = 0
        for s in range(0, n, 1 << 24):
            t += int((mi.splitmix64(1 << 24, 4 + r, s) >> np.uint64(33)).sum())
        sums.append(t)
    for p in (1, 2):
        assert sum(x["sum"] for x in d[str(p)]) == sum(sums[:p]), p


def test_config_digests_match_survey():
    """tests/golden/config_digests.json (make_config_digests.py: oracle only):
    first / last sorted key (and payload) of C1-C4 equal the survey's
    independent numpy values (SURVEY.md §8(c) golden values)."""
    with open(os.path.join(GOLDEN, "config_digests.json")) as f:
        g = json.load(f)["configs"]
    for name, exp in SURVEY.items():
        d = g[name]
        assert d["n"] == mi.CONFIGS[name]["n"], name
        assert d["first"] == exp["sorted_at"][0] and d["last"] == exp["sorted_at"][-1], name
        if "payload_at" in exp:
            assert d["vals_first"] == exp["payload_at"][0], name
            assert d["vals_last"] == exp["payload_at"][-1], name
        assert len(d["keys_sha256"]) == 64


def test_oracle_live_c1_matches_survey(orc):
    k, _ = mi.config_input("C1")
    s = orc.sort(k)
    n = k.size
    assert [int(s[p]) for p in (0, n // 4, n // 2, 3 * n // 4, n - 1)] == SURVEY["C1"]["sorted_at"]
    assert orc.check(k, s) == 0
    assert np.array_equal(s, np.sort(k, kind="stable"))


@pytest.mark.parametrize("dtype", [np.int32, np.uint64])
def test_segmented_definition(orc, dtype):
    """Batched sort (f3): the oracle's per-segment sort equals the library
    routine numpy.lexsort by (segment id, key) -- stable, so equal keys of a
    segment keep their input order -- including empty and 1-element segments."""
    rng = np.random.default_rng(7)
    lens = np.concatenate([[0, 1, 2, 0, 3], rng.integers(0, 70, 400), [500, 0]])
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(off[-1])
    k = rng.integers(0, 9, n).astype(dtype)  # heavy duplicates: stability is visible
    v = np.arange(n, dtype=np.uint32)
    seg = np.repeat(np.arange(lens.size), lens)
    perm = np.lexsort((k, seg))  # last key primary; lexsort is stable
    ok, ov = orc.sort_segmented(k, off, v)
    assert np.array_equal(ok, k[perm]) and np.array_equal(ov, v[perm])
    assert np.array_equal(orc.sort_segmented(k, off), k[perm])
    # one segment = the plain sort
    assert np.array_equal(orc.sort_segmented(k, [0, n]), orc.sort(k))


def test_tree_rank_order_closed_form(orc):
    """For p = 2^k the paper's tree leaves ties in bit-reversed rank
    order (SURVEY ledger L11); p = 1 and p = 2 are the identity."""
    assert orc.tree_rank_order(1) == [0]
    assert orc.tree_rank_order(2) == [0, 1]
    assert orc.tree_rank_order(4) == [0, 2, 1, 3]
    for k in range(1, 7):
        p = 1 << k
        rev = [int(format(r, f"0{k}b")[::-1], 2) for r in range(p)]
        assert orc.tree_rank_order(p) == rev
    # non powers of two: a permutation of the ranks, rank 0 first
    for p in (3, 5, 6, 7, 12):
        o = orc.tree_rank_order(p)
        assert sorted(o) == list(range(p)) and o[0] == 0


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8])
def test_sort_tree_is_stable_sort_in_tree_order(orc, p):
    """The literal tree of merges equals numpy's stable argsort of the shards
    concatenated in tree order (a library routine), payload = (rank, index)."""
    rng = np.random.default_rng(p)
    shards = [rng.integers(0, 6, int(rng.integers(0, 40))).astype(np.int32) for _ in range(p)]
    vals = [(np.uint32(r) << np.uint32(16)) + np.arange(s.size, dtype=np.uint32)
            for r, s in enumerate(shards)]
    ok, ov = orc.sort_tree(shards, vals)
    order = orc.tree_rank_order(p)
    cat = np.concatenate([shards[r] for r in order])
    catv = np.concatenate([vals[r] for r in order])
    perm = np.argsort(cat, kind="stable")
    assert np.array_equal(ok, cat[perm]) and np.array_equal(ov, catv[perm])
    assert np.array_equal(orc.sort_tree(shards), cat[perm])
