"""Parity of the in-kernel outlier route (-m gpu): nearly sorted keys
(k-exchange; configs[1](c) "n/100 random pair swaps") inside the
resident launch (resident.cuh ResOut): the endpoints of every descent
 are extracted per tile, bucketed by splitters taken from the
sorted remainder and merged back per bucket, bit-exact against
the CPU oracle.  The hand-offs to the host's outlier rounds (an unsorted tile,
a tile boundary out of order, a full bucket) leave the keys untouched and are
exercised with inputs built to trigger each one."""
import numpy as np
import pytest
import torch

import oracle
import paper_1609_04471_b200 as sr
from workloads import gen

pytestmark = pytest.mark.gpu

TO32 = 8192  # ResOut<int32_t>::TO (outlier tile)
OCAP32 = 256  # ResOut<int32_t>::OCAP (outliers per bucket)
MAXN32, MAXN64 = 768 * 4096, 384 * 2048  # ResOut<K>::MAXN (the route's n range)


@pytest.fixture(autouse=True)
def _reset():
    yield
    sr.set_option(sr.OPT_FORCE_ROUTE, 0)
    sr.set_option(sr.OPT_OUTLIER_ROUTE, 1)
    sr.set_option(sr.OPT_RESIDENT, 1)


def check(k):
    d = torch.from_numpy(k.copy()).cuda()
    sr.sort_keys(d)
    torch.cuda.synchronize()
    e = oracle.sort_keys(k)
    got = d.cpu().numpy()
    assert np.array_equal(got, e), f"n={k.size}: first mismatch at {int(np.argmax(got != e))}"
    return sr.last_plan()


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("n", [8193, 65_537, 300_007, 1_000_000, 2_000_000, 4_194_304])
def test_res_outlier_c2_nearly(n, dtype):
    """configs[1](c) at every resident size: one launch when the route holds."""
    for inst in range(2):
        k = gen.make("nearly", n, dtype, config=1, instance=inst)
        p = check(k)
        # the in-kernel route's range (within the resident range, 2.36M keys)
        if p["route_name"] == "outlier" and n <= (MAXN32 if dtype == np.int32 else MAXN64):
            assert p["launches"] == 1, p


@pytest.mark.parametrize("swaps", [1, 10, 100, 1000, 20_000, 60_000])
def test_res_outlier_swap_counts(swaps):
    n = 2_000_000
    p = check(gen.swaps(n, swaps, np.int32, 900 + swaps))
    assert p["route_name"] in ("outlier", "partition"), p
    if swaps <= 20_000:
        assert p["route_name"] == "outlier" and p["launches"] == 1, p


def test_res_outlier_clustered_swaps():
    """Swaps of neighbouring positions and chains through shared positions:
    the per-tile iteration removes more than the descent endpoints."""
    n = 2_000_000
    rng = np.random.default_rng(11)
    for trial in range(4):
        a = np.arange(n, dtype=np.int32)
        for _ in range(3000):
            p = int(rng.integers(0, n - 8))
            q = p + int(rng.integers(1, 6)) if trial % 2 == 0 else int(rng.integers(0, n))
            a[p], a[q] = a[q], a[p]
        check(a)


def test_res_outlier_tile_edges():
    """Swaps at and around the outlier tiles' boundaries (the halo keys)."""
    n = 1_500_000
    a = np.arange(n, dtype=np.int32)
    for t in range(TO32, n - 2, TO32):
        for d in (-1, 0, 1):
            p = t + d
            q = (p * 7919) % n
            a[p], a[q] = a[q], a[p]
    check(a)


def test_res_outlier_full_bucket_hands_off():
    """2000 outliers of one value fill one bucket past OCAP (512): the host's rounds
    sort from the untouched keys."""
    n = 2_000_000
    a = np.arange(n, dtype=np.int32)
    pos = np.linspace(1000, n - 1000, 2000).astype(np.int64)
    a[pos] = 5
    p = check(a)
    assert p["launches"] > 1, p  # not finished in the one launch


def test_res_outlier_boundary_out_of_order_hands_off():
    """A step down exactly at an outlier tile boundary: every tile's kept keys
    are sorted but the remainder is not (forced route)."""
    n = 1_000_000
    a = np.arange(n, dtype=np.int32)
    a[8 * TO32:] -= 1000
    sr.set_option(sr.OPT_FORCE_ROUTE, sr.ROUTE_OUTLIER)
    p = check(a)
    assert p["launches"] > 1, p


def test_res_outlier_equal_keys():
    """Nearly sorted with long runs of equal keys (ties between the remainder
    and the outliers: the remainder wins)."""
    n = 2_000_000
    a = (np.arange(n, dtype=np.int64) // 37).astype(np.int32)
    rng = np.random.default_rng(3)
    for _ in range(5000):
        p, q = int(rng.integers(0, n)), int(rng.integers(0, n))
        a[p], a[q] = a[q], a[p]
    check(a)
    b = np.repeat(np.arange(50, dtype=np.int32), n // 50)
    b[::4001] = 17
    check(b)


def test_res_outlier_extreme_values():
    n = 1_000_003
    a = np.arange(n, dtype=np.int32) - n // 2
    rng = np.random.default_rng(9)
    idx = rng.integers(0, n, 3000)
    a[idx[:1000]] = np.iinfo(np.int32).max
    a[idx[1000:2000]] = np.iinfo(np.int32).min
    check(a)
    a64 = np.arange(n, dtype=np.int64) * (1 << 30)
    a64[idx[:100]] = np.iinfo(np.int64).min
    check(a64)


def test_res_outlier_disabled():
    sr.set_option(sr.OPT_OUTLIER_ROUTE, 0)
    p = check(gen.make("nearly", 2_000_000, np.int32, config=1))
    assert p["route_name"] != "outlier"


def test_res_outlier_c2_instances_stay_in_kernel():
    """The bench's C2 nearly instances: clusters of exchanges that straddle a
    tile boundary are resolved by trimming the boundary (no host hand-off)."""
    n = 2_000_000
    in_kernel = 0
    for inst in range(20):
        p = check(gen.make("nearly", n, np.int32, config=1, instance=inst))
        assert p["route_name"] == "outlier", p
        in_kernel += p["launches"] == 1
    assert in_kernel == 20, in_kernel


def test_res_outlier_boundary_trim():
    """Exchanges chained through both sides of every outlier tile boundary."""
    n = 1_200_000
    a = np.arange(n, dtype=np.int32)
    for t in range(TO32, n - 64, TO32):
        a[t - 2], a[t + 1] = a[t + 1], a[t - 2]
        a[t - 1], a[t + 3] = a[t + 3], a[t - 1]
        a[t - 5], a[t] = a[t], a[t - 5]
    sr.set_option(sr.OPT_FORCE_ROUTE, sr.ROUTE_OUTLIER)  # (auto: the k-distance route takes it)
    p = check(a)
    assert p["route_name"] == "outlier" and p["launches"] == 1, p
