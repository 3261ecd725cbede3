"""The k-distance route (distance.cuh): inputs whose keys
lie fewer than 512 positions from their sorted places (Table 1's
nearly sorted class is 256-distance) are proven so by the
presortedness scan and sorted by window sorts + window merges.  Every case is
compared bit-exact with the oracle; the route is asserted where the bound holds
(and asserted NOT taken where it does not)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1609_04471_b200 as sr
from workloads import gen

pytestmark = pytest.mark.gpu


def _dist(n, k, dt, seed):
    """gen.distance(n, k, dt, seed), built on the device (sr_generate is
    bit-identical to workloads/gen.py, tests/test_gpu_generate.py; the Python
    loop takes minutes at 16M keys)."""
    t = torch.empty(n, dtype=torch.int32 if np.dtype(dt) == np.int32 else torch.int64, device="cuda")
    sr.generate(t, "distance", seed, k)
    return t.cpu().numpy()


def _sort(k):
    d = torch.from_numpy(k.copy()).cuda()
    sr.sort_keys(d)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), oracle.sort_keys(k))
    return sr.last_plan()["route_name"]


@pytest.mark.parametrize("dt", [np.int32, np.int64])
@pytest.mark.parametrize("n", [300_007, 2_000_000, 3_000_001, 16_777_216])
def test_distance256_routed_and_exact(dt, n):
    assert _sort(_dist(n, 256, dt, gen.seed_for(1, gen.ORDERS["distance256"], 0))) == "distance"


@pytest.mark.parametrize("dt", [np.int32, np.int64])
@pytest.mark.parametrize("k", [1, 31, 255, 256, 400])
@pytest.mark.parametrize("n", [100_003, 2_500_001])
def test_distance_k_exact(dt, k, n):
    # blocks of k + 1 <= 257 keys always pass the subtile test (no block reaches
    # both subtile q and subtile q + 2 of 256 keys); k = 400 may or may not
    a = _dist(n, k, dt, gen.seed_for(9, 18, k))
    route = _sort(a)
    if k <= 256:
        assert route == "distance"


@pytest.mark.parametrize("n", [200_000, 3_000_000])
def test_distance_bound_exceeded_not_routed(n):
    a = _dist(n, 1500, np.int32, gen.seed_for(9, 18, 1500))  # displacements up to 1500
    assert _sort(a) != "distance"


@pytest.mark.parametrize("n", [65_537, 1_048_577, 4_194_305])
def test_distance_ties_and_ragged(n):
    # few distinct values, locally shuffled: ties across subtile boundaries
    base = (np.arange(n, dtype=np.int64) // 700).astype(np.int32)
    rng = np.random.default_rng(n)
    a = base.copy()
    for s in range(0, n, 200):  # blocks of 200 <= 257
        rng.shuffle(a[s:s + 200])
    assert _sort(a) == "distance"


def test_distance_adjacent_swaps_exact():
    n = 3_000_000
    a = np.arange(n, dtype=np.int32)
    i = np.arange(0, n - 1, 97)
    a[i], a[i + 1] = a[i + 1].copy(), a[i].copy()
    _sort(a)


def test_distance_route_disabled():
    sr.set_option(sr.OPT_DISTANCE_ROUTE, 0)
    try:
        assert _sort(_dist(2_000_000, 256, np.int32, 5)) != "distance"
    finally:
        sr.set_option(sr.OPT_DISTANCE_ROUTE, 1)
