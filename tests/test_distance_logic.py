"""CPU check of the k-distance route's logic (distance.cuh, presort.cuh
tile_mm_finish), at reduced sizes: the subtile test (max of subtile q <= min of
subtile q+2 for all q) implies every displacement is < 2 S (S = subtile), and
then sorting windows [2jT, 2jT+2T) followed by merging windows
[(2j+1)T, (2j+1)T+2T), T = 2 S, yields the sorted array.  Pure
numpy on small arrays; np.sort is only used to define the expected output."""
import numpy as np
import pytest

pytestmark = []


def subtile_test(a, S):
    q = -(-len(a) // S)
    mn = np.array([a[i * S:(i + 1) * S].min() for i in range(q)])
    mx = np.array([a[i * S:(i + 1) * S].max() for i in range(q)])
    return bool(np.all(mx[:-2] <= mn[2:])) if q > 2 else True


def two_pass(a, T):
    a = a.copy()
    for s in range(0, len(a), 2 * T):
        a[s:s + 2 * T] = np.sort(a[s:s + 2 * T])
    for s in range(T, len(a), 2 * T):
        w = a[s:s + 2 * T]
        if len(w) > T:  # a merge of two sorted halves
            a[s:s + 2 * T] = np.sort(w)
    return a


def k_distance(n, k, rng, values=None):
    a = np.arange(n) if values is None else values.copy()
    for s in range(0, n, k + 1):
        seg = a[s:s + k + 1]
        rng.shuffle(seg)
    return a


@pytest.mark.parametrize("S", [2, 4, 8])
def test_subtile_test_bounds_displacement(S):
    rng = np.random.default_rng(S)
    for _ in range(300):
        n = int(rng.integers(1, 200))
        a = rng.integers(0, 40, n)
        # random local perturbation of a sorted array
        a = np.sort(a)
        for _ in range(int(rng.integers(0, 6))):
            i = int(rng.integers(0, n))
            j = min(n - 1, max(0, i + int(rng.integers(-3 * S, 3 * S))))
            a[i], a[j] = a[j], a[i]
        if not subtile_test(a, S):
            continue
        # stable ranks: displacement < 2 S for every element
        order = np.argsort(a, kind="stable")
        rank = np.empty(n, dtype=np.int64)
        rank[order] = np.arange(n)
        assert np.all(np.abs(rank - np.arange(n)) < 2 * S)
        assert np.array_equal(two_pass(a, 2 * S), np.sort(a))


@pytest.mark.parametrize("S", [2, 4, 16])
def test_k_distance_blocks_pass_and_sort(S):
    # the scan's test accepts PAPER.md:84's k-distance construction for k <= S
    # (kDSub = 256: Table 1's 256-distance class)
    rng = np.random.default_rng(100 + S)
    for k in range(0, S + 1):  # blocks of k + 1 <= S + 1 keys never reach both subtile q and subtile q + 2
        for n in (1, 5, 2 * S + 1, 7 * S + 3, 64 * S):
            a = k_distance(n, k, rng)
            assert subtile_test(a, S)
            assert np.array_equal(two_pass(a, 2 * S), np.arange(n))


def test_k_above_subtile_can_fail_the_test():
    # a block of S + 2 keys can reach subtiles q and q + 2 (then the route is not taken)
    S = 4
    a = np.arange(16)
    a[2], a[2 + S + 1] = a[2 + S + 1], a[2]  # within one block of S + 2, positions 2 and 7
    assert not subtile_test(a, S) or np.array_equal(two_pass(a, 2 * S), np.sort(a))


def test_two_pass_needs_the_bound():
    # a displacement of 2 T breaks two passes: the test must reject such inputs
    T = 4
    a = np.arange(32)
    a[0], a[2 * T] = a[2 * T], a[0]
    assert not np.array_equal(two_pass(a, T), np.arange(32))
    assert not subtile_test(a, T // 2)


def test_ties_across_subtiles():
    rng = np.random.default_rng(7)
    S = 4
    for _ in range(200):
        n = int(rng.integers(10, 120))
        a = k_distance(n, int(rng.integers(0, S + 1)), rng, values=np.arange(n) // int(rng.integers(1, 6)))
        assert subtile_test(a, S)
        assert np.array_equal(two_pass(a, 2 * S), np.sort(a))
