"""Pins for the CPU oracle (-m "not gpu").

Each check ties the oracle to something other than itself: brute force over
tiny inputs, the stable-rank definition, a library routine for
special cases (Python's stable `sorted`, numpy searchsorted), closed forms of
the paper's constructions, and the paper's worked example
 stored under tests/golden/.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from workloads import gen


def _golden(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- brute force

@pytest.mark.parametrize("n", range(0, 9))
def test_all_permutations_sort_to_identity(n):
    """north star: brute force over all permutations of n <= 8."""
    target = np.arange(n, dtype=np.int32)
    for p in itertools.permutations(range(n)):
        out = oracle.sort_keys(np.array(p, dtype=np.int32))
        assert np.array_equal(out, target), p


def _stable_positions(keys):
    """position(i) = #{j: k_j < k_i} + #{j < i: k_j = k_i}."""
    n = len(keys)
    return [sum(1 for j in range(n) if keys[j] < keys[i] or (keys[j] == keys[i] and j < i)) for i in range(n)]


@pytest.mark.parametrize("n", range(1, 9))
def test_all_ternary_sequences_stable_rank(n):
    """Every sequence over {0,1,2} of length <= 8 with payload = index: the
    oracle's output places element i at its stable rank."""
    for seq in itertools.product(range(3), repeat=n):
        k = np.array(seq, dtype=np.int64)
        ok, ov = oracle.sort_pairs(k, np.arange(n, dtype=np.uint32))
        pos = _stable_positions(seq)
        expect_v = np.empty(n, np.uint32)
        for i, p in enumerate(pos):
            expect_v[p] = i
        assert np.array_equal(ov, expect_v), seq
        assert np.array_equal(ok, k[expect_v]), seq


@pytest.mark.parametrize("n", range(1, 6))
def test_ternary_brute_force_orderings(n):
    """Enumerate all n! orderings; exactly one is key-sorted with increasing
    index among equal keys, and it is the oracle's output (north star)."""
    for seq in itertools.product(range(3), repeat=n):
        ok, ov = oracle.sort_pairs(np.array(seq, np.int32), np.arange(n, dtype=np.uint32))
        good = [perm for perm in itertools.permutations(range(n))
                if all(seq[perm[t]] < seq[perm[t + 1]] or (seq[perm[t]] == seq[perm[t + 1]] and perm[t] < perm[t + 1])
                       for t in range(n - 1))]
        assert len(good) == 1
        assert list(ov) == list(good[0])


# ---------------------------------------------------------------- cross-checks

def _insertion_sort_pairs(keys, vals):
    """Hand-written stable insertion sort: shift while a[j-1].key > x.key (strict)."""
    k = list(keys)
    v = list(vals)
    for i in range(1, len(k)):
        xk, xv = k[i], v[i]
        j = i
        while j > 0 and k[j - 1] > xk:
            k[j], v[j] = k[j - 1], v[j - 1]
            j -= 1
        k[j], v[j] = xk, xv
    return k, v


ORDERS_SMALL = ["random", "reversed", "nearly", "few_unique", "organ_pipe", "extremes", "all_equal", "runs1024"]


@pytest.mark.parametrize("order", ORDERS_SMALL)
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_vs_insertion_sort(order, dtype):
    n = 1500
    k = gen.make(order, n, dtype, config=90)
    v = np.arange(n, dtype=np.uint32)
    ek, ev = _insertion_sort_pairs(k.tolist(), v.tolist())
    ok, ov = oracle.sort_pairs(k, v)
    assert ok.tolist() == ek and ov.tolist() == ev
    assert oracle.sort_keys(k).tolist() == ek


@pytest.mark.parametrize("order", ORDERS_SMALL + ["few100", "alternating", "sharp_teeth"])
def test_vs_library_stable_sort(order):
    """Python's sorted() is a stable library sort: a special case reference."""
    n = 100_003
    k = gen.make(order, n, np.int32, config=91)
    v = np.arange(n, dtype=np.uint32)
    idx = sorted(range(n), key=lambda i: int(k[i]))
    ok, ov = oracle.sort_pairs(k, v)
    assert np.array_equal(ov, np.array(idx, np.uint32))
    assert np.array_equal(ok, k[idx])


def test_sortedness_and_multiset_by_counting():
    n = 1_000_000
    k = gen.make("random", n, np.int32, config=92)
    out = oracle.sort_keys(k)
    assert np.all(out[:-1] <= out[1:])
    u1, c1 = np.unique(k, return_counts=True)
    u2, c2 = np.unique(out, return_counts=True)
    assert np.array_equal(u1, u2) and np.array_equal(c1, c2)


# ---------------------------------------------------------------- closed forms

@pytest.mark.parametrize("order", ["reversed", "nearly", "swaps_1e4", "swaps_1e1", "runs1024", "sharp_teeth", "sorted"])
def test_constructions_sort_to_ramp(order):
    """Reversed, k-exchange, shuffled blocks, sharp teeth are permutations of
    0..n-1 (constructions from a sorted list)."""
    n = 300_007
    k = gen.make(order, n, np.int32, config=93)
    assert np.array_equal(oracle.sort_keys(k), np.arange(n, dtype=np.int32))


def test_few_unique_closed_form():
    n = 200_000
    k = gen.make("few_unique", n, np.int32, config=94)
    vals = sorted(set(k.tolist()))
    assert len(vals) == 10
    expect = np.concatenate([np.full(int((k == v).sum()), v, np.int32) for v in vals])
    assert np.array_equal(oracle.sort_keys(k), expect)


def test_pairs_index_payload_invariants():
    """configs[3]: payload = original index pins the stable output completely."""
    n = 300_000
    k = gen.make("few100", n, np.int32, config=95)
    ok, ov = oracle.sort_pairs(k, gen.index_payload(n))
    assert np.array_equal(np.sort(ov), np.arange(n, dtype=np.uint32))
    assert np.array_equal(ok, k[ov])
    same = ok[:-1] == ok[1:]
    assert np.all(ok[:-1] <= ok[1:])
    assert np.all(ov[:-1][same] < ov[1:][same])


# ---------------------------------------------------------------- golden fixtures

def test_F1_worked_example(golden_dir):
    g = _golden(golden_dir, "F1_worked_example.json")
    k = np.array(g["keys"], np.int32)
    assert oracle.descents(k) == g["descents"] == g["run"] - 1
    asc = oracle.asc_runs(k)
    assert list(asc[0]) == g["asc_run_first"]
    desc = oracle.desc_runs(k, strict=False)
    assert list(desc[-1]) == g["desc_run_last_start_len"]
    r = k.copy()
    oracle.reverse(r, 5, 16)
    assert r.tolist() == g["after_reversal_of_5_16"]
    assert oracle.sort_keys(k).tolist() == g["sorted"]
    a = np.array(g["merge_A"], np.int32)
    b = np.array(g["merge_B"], np.int32)
    for d, i in g["merge_path"].items():
        assert oracle.merge_path(a, b, int(d)) == i
    assert oracle.merge(a, b).tolist() == g["sorted"]


@pytest.mark.parametrize("name", ["F2_pairs_find_run.json", "F3_organ_pipe_ties.json", "F6_all_equal_pairs.json"])
def test_pair_fixtures(golden_dir, name):
    g = _golden(golden_dir, name)
    ok, ov = oracle.sort_pairs(np.array(g["keys"], np.int32), np.array(g["vals"], np.uint32))
    assert ok.tolist() == g["sorted_keys"] and ov.tolist() == g["sorted_vals"]
    if "asc_runs" in g:
        k = np.array(g["keys"], np.int32)
        assert [list(r) for r in oracle.asc_runs(k)] == g["asc_runs"]
        assert [list(r) for r in oracle.desc_runs(k, strict=True)] == g["desc_runs_strict"]
        assert [list(r) for r in oracle.desc_runs(k, strict=False)] == g["desc_runs_nonstrict"]


@pytest.mark.parametrize("name", ["F4_bsd_adversarial.json", "F5_signed_extremes.json"])
def test_key_fixtures(golden_dir, name):
    g = _golden(golden_dir, name)
    k = np.array(g["keys"], np.int32)
    assert oracle.sort_keys(k).tolist() == g["sorted"]
    if "descents" in g:
        assert oracle.descents(k) == g["descents"]
    assert gen.bsd_adversarial(3, np.int32).tolist() == _golden(golden_dir, "F4_bsd_adversarial.json")["keys"]


def test_F7_reversed(golden_dir):
    for n in _golden(golden_dir, "F7_reversed.json")["sizes"]:
        k = gen.reversed_ramp(n, np.int32)
        assert oracle.descents(k) == n - 1  # Run(A) = n
        assert oracle.desc_runs(k, strict=True) == [(0, n)]
        assert np.array_equal(oracle.sort_keys(k), np.arange(n, dtype=np.int32))


# ---------------------------------------------------------------- presortedness

@pytest.mark.parametrize("seed", range(20))
def test_runs_are_maximal_monotone_partitions(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 200))
    k = rng.integers(0, 4, n).astype(np.int32)
    for runs, ok_pair in [(oracle.asc_runs(k), lambda x, y: x <= y),
                          (oracle.desc_runs(k, strict=False), lambda x, y: x >= y),
                          (oracle.desc_runs(k, strict=True), lambda x, y: x > y)]:
        pos = 0
        for s, l in runs:
            assert s == pos and l >= 1
            seg = k[s:s + l].tolist()
            assert all(ok_pair(seg[t], seg[t + 1]) for t in range(l - 1))
            if s + l < n:  # maximal: cannot extend by one
                assert not ok_pair(int(k[s + l - 1]), int(k[s + l]))
            pos += l
        assert pos == n
    assert len(oracle.asc_runs(k)) == oracle.descents(k) + 1  # Run(A) = D + 1


def test_even_teeth_mono_equals_k():
    """for k <= n/3 a k-even teeth has Mono = k; with distinct
    values inside a tooth, its maximal monotone runs alternate direction."""
    k = gen.even_teeth(1200, 8, np.int32)
    d = oracle.desc_runs(k, strict=True)
    a = oracle.asc_runs(k)
    # 4 strictly descending teeth of 150; 4 ascending teeth that absorb the
    # equal neighbours at tooth boundaries (1,1 and 150,150), so 150..152 long
    assert sum(1 for _, l in d if l == 150) == 4
    assert sorted(l for _, l in a if l >= 150) == [151, 152, 152, 152]


# ---------------------------------------------------------------- merge / merge path

@pytest.mark.parametrize("seed", range(30))
def test_merge_is_stable_union(seed):
    rng = np.random.default_rng(seed)
    a = np.sort(rng.integers(0, 5, int(rng.integers(0, 40)))).astype(np.int32)
    b = np.sort(rng.integers(0, 5, int(rng.integers(0, 40)))).astype(np.int32)
    va = np.arange(a.size, dtype=np.uint32)
    vb = np.arange(a.size, a.size + b.size, dtype=np.uint32)
    out, vout = oracle.merge(a, b, va, vb)
    # concatenation sorted stably by key == stable merge with A winning ties
    cat = np.concatenate([a, b])
    idx = sorted(range(cat.size), key=lambda i: int(cat[i]))
    assert out.tolist() == cat[idx].tolist() and vout.tolist() == idx


@pytest.mark.parametrize("seed", range(30))
def test_merge_path_split_invariant(seed):
    """For every diagonal d the split i (j = d - i) satisfies A[i-1] <= B[j]
    and B[j-1] < A[i]: the set of first-d outputs (A wins ties)."""
    rng = np.random.default_rng(100 + seed)
    a = np.sort(rng.integers(0, 6, int(rng.integers(0, 25)))).astype(np.int64)
    b = np.sort(rng.integers(0, 6, int(rng.integers(0, 25)))).astype(np.int64)
    for d in range(a.size + b.size + 1):
        i = oracle.merge_path(a, b, d)
        j = d - i
        assert 0 <= i <= a.size and 0 <= j <= b.size
        if i > 0 and j < b.size:
            assert a[i - 1] <= b[j]
        if j > 0 and i < a.size:
            assert b[j - 1] < a[i]


# ---------------------------------------------------------------- partition pieces

@pytest.mark.parametrize("seed", range(10))
def test_classify_matches_searchsorted(seed):
    rng = np.random.default_rng(seed)
    keys = rng.integers(-50, 50, 5000).astype(np.int32)
    spl = np.unique(rng.integers(-60, 60, int(rng.integers(1, 40)))).astype(np.int32)
    eq = rng.integers(0, 2, spl.size).astype(np.uint8)
    bins = oracle.classify(keys, spl, eq)
    i = np.searchsorted(spl, keys, side="left")  # #{t < x}
    hit = (i < spl.size) & (spl[np.minimum(i, spl.size - 1)] == keys) & (eq[np.minimum(i, spl.size - 1)] == 1)
    assert np.array_equal(bins, 2 * i + hit)
    # bucket order is key order: concatenating buckets in id order is sorted by bucket
    assert np.all(np.diff(bins[np.argsort(keys, kind="stable")]) >= 0)


@pytest.mark.parametrize("seed", range(10))
def test_classify_with_repeated_splitters(seed):
    """Repeated splitter values: every key equal to a repeated splitter goes to
    the first copy (lower_bound); the buckets between the copies stay empty."""
    rng = np.random.default_rng(50 + seed)
    keys = rng.integers(-20, 20, 5000).astype(np.int64)
    spl = np.sort(rng.integers(-25, 25, int(rng.integers(1, 60)))).astype(np.int64)
    vals, first = np.unique(spl, return_index=True)
    flag_of = {int(v): int(rng.integers(0, 2)) for v in vals}
    eq = np.array([flag_of[int(v)] for v in spl], np.uint8)
    bins = oracle.classify(keys, spl, eq)
    i = np.searchsorted(spl, keys, side="left")
    hit = (i < spl.size) & (spl[np.minimum(i, spl.size - 1)] == keys) & (eq[np.minimum(i, spl.size - 1)] == 1)
    assert np.array_equal(bins, 2 * i + hit)
    used = set(bins.tolist())
    for j in range(1, spl.size):  # no key lands between two copies of a value
        if spl[j] == spl[j - 1]:
            assert 2 * j not in used and 2 * j + 1 not in used


def test_stable_partition_matches_stable_library_sort():
    rng = np.random.default_rng(7)
    n = 20000
    keys = rng.integers(0, 1000, n).astype(np.int64)
    bins = rng.integers(0, 37, n).astype(np.int32)
    ok, ov, counts = oracle.stable_partition(bins, 37, keys, np.arange(n, dtype=np.uint32))
    idx = sorted(range(n), key=lambda t: int(bins[t]))
    assert ov.tolist() == idx and ok.tolist() == keys[idx].tolist()
    assert counts.tolist() == np.bincount(bins, minlength=37).tolist()


@pytest.mark.parametrize("order", ["random", "few_unique", "organ_pipe", "all_equal", "nearly"])
def test_splitters_properties(order):
    n = 200_000
    k = gen.make(order, n, np.int32, config=96)
    B, o = 256, 8
    spl, eq = oracle.splitters(k, 0, n, B, o)
    S = B * o
    assert spl.size == B - 1
    assert np.all(np.diff(spl.astype(np.int64)) >= 0)  # non-decreasing (repeats delimit empty buckets)
    pos = [oracle.sample_pos(0, n, S, t) for t in range(S)]
    for t, p in enumerate(pos):  # one sample per stratum
        assert (t * n) // S <= p < ((t + 1) * n) // S
    smp = np.sort(k[pos])  # library sort of the sample: order statistics
    cand = [smp[((j + 1) * S) // B] for j in range(B - 1)]
    assert spl.tolist() == [int(c) for c in cand]
    for t, f in zip(spl, eq):
        assert f == (int((smp == t).sum()) > 2)  # gamma = 2
    if order == "few_unique":  # all 10 values become equality splitters
        assert len(set(spl.tolist())) == 10 and eq.all()
    if order == "all_equal":
        assert len(set(spl.tolist())) == 1 and eq.all()


def test_count_and_stable_rank():
    k = np.array([5, 3, 5, 1, 3, 5], np.int64)
    assert oracle.count(k, 3) == (1, 3)
    assert oracle.count(k, 5) == (3, 6)
    assert [oracle.stable_rank(k, i) for i in range(6)] == _stable_positions(k.tolist())


# ---- floating-point keys: IEEE 754 totalOrder --------

def test_float_golden_total_order(golden_dir):
    """F8: hand-ordered special values, keys and stable payloads (golden fixture)."""
    d = _golden(golden_dir, "F8_float_total_order.json")
    k = np.array([int(x, 16) for x in d["input_bits"]], np.uint32).view(np.float32)
    exp = np.array([int(x, 16) for x in d["expected_bits"]], np.uint32)
    assert np.array_equal(oracle.sort_keys(k).view(np.uint32), exp)
    kk, vv = oracle.sort_pairs(k, np.array(d["pairs_vals"], np.uint32))
    assert np.array_equal(kk.view(np.uint32), exp)
    assert vv.tolist() == d["expected_vals"]
    # the same special values as float64
    k64 = k.astype(np.float64)  # NaN payloads widen; signs, zeros, infinities keep their order
    o64 = oracle.sort_keys(k64)
    assert np.isnan(o64[:3]).all() and np.signbit(o64[:3]).all() and np.isnan(o64[-3:]).all()
    assert o64[3] == -np.inf and o64[-4] == np.inf


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_float_finite_matches_numpy(dtype):
    """Finite keys without zeros: totalOrder is numeric order (numpy's sort)."""
    k = gen.make_float("funiform", 5000, dtype, config=97) - dtype(0.5)
    k = k[k != 0]
    assert np.array_equal(oracle.sort_keys(k), np.sort(k))
    b = gen.make_float("fbits", 5000, dtype, config=97)
    b = b[np.isfinite(b) & (b != 0)]
    assert np.array_equal(oracle.sort_keys(b), np.sort(b))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_float_random_bits_properties(dtype):
    """Random bit patterns (all classes): a permutation of the input bits,
    negative signs first, numeric order inside each sign class, NaNs outside."""
    it = np.uint32 if dtype == np.float32 else np.uint64
    k = gen.make_float("fbits", 20000, dtype, config=98)
    k[:64] = gen.make_float("fspecial", 64, dtype, config=98)
    o = oracle.sort_keys(k)
    assert np.array_equal(np.sort(o.view(it)), np.sort(k.view(it)))
    sb = np.signbit(o)
    assert not np.any(sb[1:] & ~sb[:-1])  # no negative after a positive
    for part in (o[sb], o[~sb]):
        fin = part[~np.isnan(part)]
        assert np.all(fin[1:] >= fin[:-1])
        nanpos = np.flatnonzero(np.isnan(part))
        if nanpos.size:  # negative NaNs lead, positive NaNs trail
            if np.signbit(part[0]):
                assert nanpos.tolist() == list(range(nanpos.size))
            else:
                assert nanpos.tolist() == list(range(part.size - nanpos.size, part.size))
    # -0 before +0, each zero class contiguous
    z = np.flatnonzero(o == 0)
    if z.size:
        zs = np.signbit(o[z])
        assert not np.any(zs[1:] & ~zs[:-1])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_float_pairs_stable(dtype):
    """Stability with ties (payload = input index): equal bit patterns keep input order."""
    it = np.uint32 if dtype == np.float32 else np.uint64
    k = gen.make_float("fspecial", 3000, dtype, config=99)
    v = np.arange(k.size, dtype=np.uint32)
    ok, ov = oracle.sort_pairs(k, v)
    assert np.array_equal(ok.view(it), k.view(it)[ov])
    same = ok.view(it)[1:] == ok.view(it)[:-1]
    assert np.all(ov[1:][same] > ov[:-1][same])
    assert np.array_equal(oracle.sort_keys(k).view(it), ok.view(it))


# ---- record keys: lexicographic order --------

@pytest.mark.parametrize("words", [1, 2, 3, 5])
@pytest.mark.parametrize("order", ["lrandom", "lprefix", "lequal", "ldup"])
def test_records_match_python_tuples(order, words):
    """Python's sorted() on tuples is a stable lexicographic sort (library routine)."""
    r = gen.make_list(order, 700, words, config=77)
    o, perm = oracle.sort_records(r, with_perm=True)
    rows = [tuple(x) for x in r.tolist()]
    exp = sorted(range(len(rows)), key=lambda i: rows[i])
    assert perm.tolist() == exp
    assert np.array_equal(o, r[exp])


def test_records_brute_force_small():
    """All 3^4 = 81 two-word records over {-1, 0, 1} in every rotation: the output
    is the unique ascending enumeration."""
    vals = [-1, 0, 1]
    allrec = np.array([(a, b) for a in vals for b in vals for _ in range(2)], np.int32)  # 18 rows, pairs of duplicates
    for rot in range(len(allrec)):
        r = np.roll(allrec, rot, axis=0)
        o, perm = oracle.sort_records(r, with_perm=True)
        assert o.tolist() == [[a, b] for a in vals for b in vals for _ in range(2)]
        for i in range(0, len(o), 2):  # stability among identical records
            assert perm[i] < perm[i + 1]


# ---- presortedness measures ---------

def _mono_dp(a):
    """Fewest contiguous monotone pieces by dynamic programming over all cut points
    (an exhaustive alternative to the oracle's greedy)."""
    n = len(a)
    def mono(s, e):
        seg = a[s:e]
        return all(x <= y for x, y in zip(seg, seg[1:])) or all(x >= y for x, y in zip(seg, seg[1:]))
    best = [0] + [n + 1] * n
    for e in range(1, n + 1):
        for s in range(e):
            if mono(s, e):
                best[e] = min(best[e], best[s] + 1)
    return best[n]


def test_measures_closed_forms():
    n = 1000
    r = oracle.measures(np.arange(n, dtype=np.int32)[::-1].copy())
    assert (r["inversions"], r["runs"], r["mono"], r["max_dis"]) == (n * (n - 1) // 2, n, 1, n - 1)
    s = oracle.measures(np.arange(n, dtype=np.int64))
    assert (s["inversions"], s["runs"], s["mono"], s["max_dis"], s["misplaced"]) == (0, 1, 1, 0, 0)
    assert oracle.measures(np.array([1, 2, 3, 3, 2, 1], np.int32))["mono"] == 2  # organ pipe
    m = 64  # k = n/2 even teeth over {1, 2}: (2,1,1,2,2,1,1,2,...), Mono = n/4 + 1
    teeth = np.array(([2, 1, 1, 2] * (m // 4)), np.int32)
    assert oracle.measures(teeth)["mono"] == m // 4 + 1
    for k in [1, 4, 16]:  # k-equal teeth: Run = Mono = k
        t = np.tile(np.arange(1, 101, dtype=np.int32), k)
        mm = oracle.measures(t)
        assert mm["runs"] == k and mm["mono"] == k
    p, q = 100, 700  # one exchange of distinct sorted values: Inv = 2 (q - p) - 1, 2 misplaced
    a = np.arange(n, dtype=np.int32)
    a[[p, q]] = a[[q, p]]
    e = oracle.measures(a)
    assert (e["inversions"], e["misplaced"], e["max_dis"]) == (2 * (q - p) - 1, 2, q - p)


def test_measures_brute_force_small():
    rng = np.random.default_rng(5)
    for n in range(1, 8):
        for _ in range(60):
            a = rng.integers(0, 3, n).astype(np.int32)
            m = oracle.measures(a)
            assert m["mono"] == _mono_dp(a.tolist())
            assert m["inversions"] == int(np.triu(a[:, None] > a[None, :], 1).sum())
            assert m["runs"] == int((a[:-1] > a[1:]).sum()) + 1
            rank = np.empty(n, np.int64)
            rank[np.argsort(a, kind="stable")] = np.arange(n)  # library stable sort
            d = np.abs(rank - np.arange(n))
            assert m["max_dis"] == int(d.max()) and m["misplaced"] == int((d != 0).sum())


def test_mono_exhaustive_three_letters():
    """Mono against the dynamic program over all cut points on EVERY sequence
    of length <= 9 over 3 letters (the definition)."""
    import itertools
    for n in range(1, 10):
        for t in itertools.product((0, 1, 2), repeat=n):
            a = np.array(t, np.int32)
            assert oracle.measures(a)["mono"] == _mono_dp(list(t)), t


@pytest.mark.parametrize("k", [1, 8, 256])
def test_measures_generated_classes(k):
    n = 20000
    dist = gen.make("distance256", n, np.int32, config=70) if k == 256 else None
    if dist is not None:  # k-distance list: Dis <= k
        assert oracle.measures(dist)["max_dis"] <= 256
    sw = gen.swaps(n, k, np.int32, gen.seed_for(70, 2, k))  # k-exchange: misplaced <= 2k, Mono <= 2k+1
    m = oracle.measures(sw)
    assert m["misplaced"] <= 2 * k and m["mono"] <= 2 * k + 1
